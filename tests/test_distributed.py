"""World-size-2/3 gloo runs of the blockwise multi-process protocol (distributed.py) on CPU.

The compute interface is the CPU one (tests/cpu_ops.py); the protocol under test is the
product's: column partition, straddling-panel gathers, factor broadcasts, A W all-gathers,
band all-gather, row-block back transformation and the ledger.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import oracle as orc


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, b, seed, skew, out, order="pipelined"):
    import torch.distributed as dist
    import sys
    sys.path.insert(0, os.getcwd())
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        from paper_2511_16174_b200 import PipelineConfig
        from paper_2511_16174_b200.distributed import run_distributed
        from tests.cpu_ops import CpuOps
        g = np.random.default_rng(seed).standard_normal((n, n))
        a = (g + g.T) / 2
        res, events, ledger, info = run_distributed(a, PipelineConfig(workers=world, b=b,
                                                                       back_skew=skew,
                                                                       order=order),
                                                    ops=CpuOps())
        from paper_2511_16174_b200.schedule import validate_trace
        validate_trace(events, world, ledger)
        out[rank] = (res.lam, res.Q, ledger.words(stage="SBR"), ledger.words(stage="BC"),
                     ledger.messages(stage="BC"), info.get("rows", info.get("cols")),
                     {k: (ledger.words(stage=k), ledger.messages(stage=k))
                      for k in ledger.stages()})
    finally:
        dist.destroy_process_group()


def _run(world, n, b, seed, skew=0.0, order="pipelined"):
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, n, b, seed, skew, out, order), nprocs=world, join=True)
    return dict(out)


@pytest.mark.parametrize("world,n,b,skew,order", [(2, 48, 8, 0.0, "pipelined"),
                                                (2, 40, 4, 0.05, "pipelined"),
                                                (3, 91, 7, 0.0, "pipelined"),
                                                (2, 150, 4, 0.0, "pipelined"),
                                                (3, 91, 7, 0.0, "conventional"),
                                                (2, 150, 4, 0.0, "conventional"),
                                                (4, 96, 8, 0.0, "pipelined"),
                                                (4, 90, 8, 0.03, "conventional"),
                                                (8, 160, 8, 0.0, "pipelined")])
def test_blockwise_protocol_matches_oracle(world, n, b, skew, order):
    out = _run(world, n, b, seed=n + world, skew=skew, order=order)
    g = np.random.default_rng(n + world).standard_normal((n, n))
    a = (g + g.T) / 2
    lam_o, _ = orc.evd(a, b, True)
    ref = out[0]
    for r in range(world):
        lam, q, sbr_words, bc_words, bc_msgs, rows, by_stage = out[r]
        # every rank returns the same full result
        np.testing.assert_array_equal(lam, ref[0])
        np.testing.assert_array_equal(q, ref[1])
        np.testing.assert_allclose(lam, lam_o, atol=10 * n * np.finfo(float).eps * np.abs(lam_o).max())
        assert orc.backward_error(a, q, lam) <= 1e-15
        assert orc.orthogonality(q) <= 1e-15
        # ledger = the reference protocol's analytic counts (tests/test_pipeline.py:103-109)
        from paper_2511_16174_b200 import comm_broadcast_words
        assert sbr_words == comm_broadcast_words(n, b)
        assert bc_words == (world - 1) * 2 * b * b and bc_msgs == world - 1
        # the whole measured ledger = the protocol's closed form (schedule.protocol_ledger)
        from paper_2511_16174_b200.schedule import protocol_ledger
        want = {}
        for (_, _, st, w) in protocol_ledger(n, b, world, True, skew):
            wd, ms = want.get(st, (0, 0))
            want[st] = (wd + w, ms + 1)
        assert by_stage == want
    rows = [out[r][5] for r in range(world)]
    assert rows[0][0] == 0 and rows[-1][1] == n
    assert all(rows[i][1] == rows[i + 1][0] for i in range(world - 1))
