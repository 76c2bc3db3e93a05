"""The blockwise multi-GPU EVD through the C++ per-rank orchestrator (csrc/dist.cu).

* run(a, PipelineConfig(workers=G)) in ONE process: G worker threads over the peer communicator
  (pevd_syevd_multi).  On a 1-GPU box the G workers share cuda:0 -- the same protocol, messages
  and arithmetic as on G GPUs.  Checked against the oracle, the measured ledger against the
  protocol's closed form, the device-timed trace against validate_trace.
* run_distributed under a 1-rank NCCL process group: the torchrun path (pevd_dist_syevd over a
  real NCCL communicator).
"""
import os
import socket

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _sym(n, seed):
    g = np.random.default_rng(seed).standard_normal((n, n))
    return (g + g.T) / 2


def _ledger_by_stage(ledger):
    return {k: (ledger.words(stage=k), ledger.messages(stage=k)) for k in ledger.stages()}


def _want_by_stage(n, b, G, vectors, skew=0.0):
    from paper_2511_16174_b200.schedule import protocol_ledger
    want = {}
    for (_, _, st, w) in protocol_ledger(n, b, G, vectors, skew):
        wd, ms = want.get(st, (0, 0))
        want[st] = (wd + w, ms + 1)
    return want


@pytest.mark.parametrize("G,n,b,order", [(2, 64, 8, "pipelined"), (2, 300, 32, "conventional"),
                                         (3, 300, 32, "pipelined"), (3, 257, 32, "sequential"),
                                         (4, 512, 32, "conventional"), (4, 200, 16, "pipelined"),
                                         (2, 400, 48, "conventional"), (3, 500, 64, "pipelined")])
def test_workers_in_one_process(G, n, b, order):
    import paper_2511_16174_b200 as pkg
    from paper_2511_16174_b200.schedule import comm_broadcast_words, validate_trace
    a = _sym(n, 11 * n + G)
    cfg = pkg.PipelineConfig(workers=G, b=b, order=order)
    res, events, ledger, counter = pkg.run(a, cfg)
    lam_o, _ = orc.evd(a, b, True)
    eps = np.finfo(float).eps
    np.testing.assert_allclose(res.lam, lam_o, atol=10 * n * eps * np.abs(lam_o).max())
    assert orc.backward_error(a, res.Q, res.lam) <= 1e-15
    assert orc.orthogonality(res.Q) <= 1e-15
    assert res.Q.flags.f_contiguous if order == "conventional" else res.Q.flags.c_contiguous
    # measured ledger == the protocol's closed form; the reference's analytic checks
    # (tests/test_pipeline.py:103-109)
    assert _ledger_by_stage(ledger) == _want_by_stage(n, b, G, True)
    assert ledger.words(stage="SBR") == comm_broadcast_words(n, b)
    assert ledger.words(stage="BC") == (G - 1) * 2 * b * b
    assert ledger.messages(stage="BC") == G - 1
    # device-timed trace: the pipeline's dependency contract, with comm spans present
    validate_trace(events, G, ledger)
    stages = {e.stage for e in events}
    assert {"SBR", "BC", "Solver", "SBR-Back", "BC-Back", "Comm"} <= stages
    assert {e.worker for e in events if e.stage == "BC"} == set(range(G))
    # executed flops were counted per stage
    for st in ("SBR", "BC", "SBR-Back", "BC-Back", "Solver"):
        assert counter.by_stage.get(st, 0) > 0, st
    # bitwise rerun determinism (tests/test_pipeline.py:86-92)
    res2, _, _, _ = pkg.run(a, cfg)
    np.testing.assert_array_equal(res.lam, res2.lam)
    np.testing.assert_array_equal(res.Q, res2.Q)


@pytest.mark.parametrize("G,n,b,order", [(3, 700, 32, "conventional"), (4, 600, 32, "pipelined"),
                                         (2, 500, 40, "sequential")])
def test_workers_with_nccl_ordering(G, n, b, order, monkeypatch):
    """PEVD_PEER_SERIAL=1 makes the in-process communicator order every operation's device
    work after the previous one's, whatever the streams -- what NCCL does to the operations of
    one communicator.  The orchestrator's stream graph (lookahead on a second stream, the
    back-transform stream, device barriers) must stay acyclic under that order, or the multi-
    process NCCL run would deadlock where this run hangs.  Same results as without it."""
    import paper_2511_16174_b200 as pkg
    a = _sym(n, 5 * n + G)
    cfg = pkg.PipelineConfig(workers=G, b=b, order=order)
    ref, _, _, _ = pkg.run(a, cfg)
    monkeypatch.setenv("PEVD_PEER_SERIAL", "1")
    res, events, ledger, _ = pkg.run(a, cfg)
    np.testing.assert_array_equal(res.lam, ref.lam)
    np.testing.assert_array_equal(res.Q, ref.Q)
    assert ledger.total_words > 0


def test_comm_overlaps_trailing_update():
    """Lookahead, from the device events: the next group's first panel is factored and its
    broadcast runs while the previous group's rank-2K trailing update (a helper-lane SBR event,
    block = rank) is still running on the same rank."""
    import paper_2511_16174_b200 as pkg
    n, b, G = 1600, 32, 2
    a = _sym(n, 1234)
    res, events, ledger, _ = pkg.run(a, pkg.PipelineConfig(workers=G, b=b, order="conventional"))
    assert orc.backward_error(a, res.Q, res.lam) <= 1e-15
    upd = [e for e in events if e.worker == -1 and e.stage == "SBR"]
    comm = [e for e in events if e.stage == "Comm"]
    assert len(upd) >= G * 2
    overlap = [(u, c) for u in upd for c in comm
               if c.worker == u.block and c.t_start < u.t_end and u.t_start < c.t_end]
    assert overlap, "no comm span overlaps a trailing update"


def test_workers_values_only():
    import paper_2511_16174_b200 as pkg
    n, b = 300, 32
    a = _sym(n, 5)
    res, events, ledger, _ = pkg.run(a, pkg.PipelineConfig(workers=3, b=b, want_vectors=False))
    assert res.Q is None and not res.vectors_computed
    lam_o, _ = orc.evd(a, b, False)
    np.testing.assert_allclose(res.lam, lam_o, atol=10 * n * np.finfo(float).eps * np.abs(lam_o).max())
    assert _ledger_by_stage(ledger) == _want_by_stage(n, b, 3, False)


def test_straddling_panels_and_skew():
    """Partitions that split SBR panels (n not a multiple of b) and a skewed back plan."""
    import paper_2511_16174_b200 as pkg
    n, b = 203, 32
    a = _sym(n, 99)
    for order in ("pipelined", "conventional"):
        cfg = pkg.PipelineConfig(workers=3, b=b, order=order, back_skew=0.05)
        res, events, ledger, _ = pkg.run(a, cfg)
        assert orc.backward_error(a, res.Q, res.lam) <= 1e-15
        assert orc.orthogonality(res.Q) <= 1e-15
        assert ledger.words(stage="SBR-panel") > 2 * sum(
            pw * pw for _, pw, _ in pkg.round_schedule(n, b))  # straddling pieces moved
        assert _ledger_by_stage(ledger) == _want_by_stage(n, b, 3, True, 0.05)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _nccl_worker(rank, world, port, n, b, order, out):
    import sys
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.getcwd())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world, device_id=torch.device("cuda", 0))
    try:
        import paper_2511_16174_b200 as pkg
        from paper_2511_16174_b200.distributed import run_distributed
        a = _sym(n, 3 * n)
        res, events, ledger, info = run_distributed(a, pkg.PipelineConfig(workers=world, b=b,
                                                                           order=order))
        out[rank] = (res.lam, res.Q, sorted({e.stage for e in events}),
                     dict(info["counter"].by_stage))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("order", ["conventional", "pipelined"])
def test_nccl_one_rank(order):
    """The torchrun path end to end with a real NCCL communicator (one rank: this box has one
    GPU, and NCCL refuses two ranks on one device)."""
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    out = mgr.dict()
    n, b = 384, 32
    mp.spawn(_nccl_worker, args=(1, _free_port(), n, b, order, out), nprocs=1, join=True)
    lam, q, stages, flops = out[0]
    a = _sym(n, 3 * n)
    lam_o, _ = orc.evd(a, b, True)
    np.testing.assert_allclose(lam, lam_o, atol=10 * n * np.finfo(float).eps * np.abs(lam_o).max())
    assert orc.backward_error(a, q, lam) <= 1e-15
    assert orc.orthogonality(q) <= 1e-15
    assert {"SBR", "BC", "Solver", "SBR-Back", "BC-Back"} <= set(stages)
    assert flops.get("SBR", 0) > 0
