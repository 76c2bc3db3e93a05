"""Time the blockwise multi-process EVD (distributed.py) with however many ranks torchrun gives
(one per GPU, NCCL); with one rank this measures the per-rank protocol path against the fused
single-GPU orchestrator (pevd_syevd_device).

    torchrun --nproc-per-node 1 --master-addr 127.0.0.1 tools/dist_probe.py 16384
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2511_16174_b200 import PipelineConfig  # noqa: E402
from paper_2511_16174_b200.distributed import run_distributed  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    g = torch.Generator(device="cuda")
    g.manual_seed(n)
    a0 = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
    a0.add_(a0.t().clone())
    a0.mul_(0.5)
    order = sys.argv[2] if len(sys.argv) > 2 else "conventional"
    cfg = PipelineConfig(workers=dist.get_world_size(), b=32, order=order)
    out = []
    for rep in range(2):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res, events, ledger, info = run_distributed(lambda c0, c1: a0[c0:c1].clone(), cfg, n=n,
                                                    gather_q=False)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        stages = {}
        for e in events:
            stages[e.stage] = stages.get(e.stage, 0) + e.duration / 1e9
        out.append({"rep": rep, "wall_s": round(dt, 3),
                    "stages_s": {k: round(v, 3) for k, v in stages.items()}})
    if dist.get_rank() == 0:
        print(json.dumps({"n": n, "world": dist.get_world_size(), "order": order, "runs": out}),
              flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
