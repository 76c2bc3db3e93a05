"""The blockwise multi-process EVD with the CUDA compute path: two ranks sharing cuda:0 over
gloo (CUDA tensors staged through the host), checked against the oracle."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, b, seed, out, order="pipelined"):
    import sys
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.getcwd())
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        import paper_2511_16174_b200 as pkg
        g = np.random.default_rng(seed).standard_normal((n, n))
        a = (g + g.T) / 2
        res, events, ledger, counter = pkg.run(a, pkg.PipelineConfig(workers=world, b=b,
                                                                     order=order))
        out[rank] = (res.lam, res.Q, ledger.words(stage="SBR"), sorted({e.stage for e in events}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,b,order", [(64, 8, "pipelined"), (300, 32, "pipelined"),
                                       (300, 32, "conventional")])
def test_two_ranks_on_device(n, b, order):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), n, b, 7 * n, out, order), nprocs=2, join=True)
    g = np.random.default_rng(7 * n).standard_normal((n, n))
    a = (g + g.T) / 2
    lam_o, _ = orc.evd(a, b, True)
    for r in range(2):
        lam, q, words, stages = out[r]
        np.testing.assert_allclose(lam, lam_o, atol=10 * n * np.finfo(float).eps * np.abs(lam_o).max())
        assert orc.backward_error(a, q, lam) <= 1e-15
        assert orc.orthogonality(q) <= 1e-15
        need = {"SBR", "BC", "Solver", "SBR-Back", "BC-Back"}
        if order != "conventional":
            need.add("FinalMultiply")
        assert need <= set(stages)
    np.testing.assert_array_equal(out[0][1], out[1][1])
