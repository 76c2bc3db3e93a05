"""The drop-in `run()` end to end at the headline size: a host numpy matrix in, (EigenResult,
events, ledger, counter) out, wall-clock through the public API, next to the
device stage times it reports.

    python tools/e2e_run.py 49152 conventional pipelined
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_16174_b200 as pkg  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 49152
    orders = sys.argv[2:] or ["conventional"]
    g = torch.Generator(device="cuda")
    g.manual_seed(n)
    a = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
    a.add_(a.t().clone())
    a.mul_(0.5)
    host = np.empty((n, n), dtype=np.float64)          # C order, as numpy makes it
    torch.from_numpy(host).copy_(a)
    del a
    torch.cuda.empty_cache()
    for order in orders:
        t0 = time.perf_counter()
        res, events, ledger, counter = pkg.run(host, pkg.PipelineConfig(workers=1, b=32,
                                                                        order=order))
        wall = time.perf_counter() - t0
        stages = {}
        for e in events:
            stages[e.stage] = stages.get(e.stage, 0.0) + e.duration / 1e9
        span = (max(e.t_end for e in events) - min(e.t_start for e in events)) / 1e9
        print(json.dumps({"n": n, "order": order, "wall_s": round(wall, 3),
                          "tflops_4n3": round(4 * n ** 3 / wall / 1e12, 3),
                          "device_span_s": round(span, 3),
                          "host_overhead_s": round(wall - span, 3),
                          "stages_s": {k: round(v, 3) for k, v in stages.items()},
                          "q_order": "C" if res.Q.flags.c_contiguous else "F",
                          "executed_macs": counter.multiply_adds}), flush=True)
        del res


if __name__ == "__main__":
    main()
