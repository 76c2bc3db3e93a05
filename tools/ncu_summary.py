"""One-screen summary of an ncu --set full report (raw metrics + SASS stall attribution)."""
import collections, csv, io, subprocess, sys

KEYS = ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__cycles_elapsed.avg.per_second", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]

def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u, v = r[0], r[1], r[2]
    d = {h[i]: (v[i], u[i]) for i in range(len(h))}
    for k in KEYS:
        if k in d:
            print(f"{k:80s} {d[k][0]:>16s} {d[k][1]}")
    st = [(k, float(d[k][0])) for k in d if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio") and d[k][0] not in ("", "0")]
    st.sort(key=lambda x: -x[1])
    print("stalls/issue:", ", ".join(f"{k.split('stalled_')[1].split('_per')[0]}={v:.2f}" for k, v in st[:8]))

def source(path, top=12):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    ci = {k: i for i, k in enumerate(h)}
    data = []
    for r in rows[2:]:
        try:
            data.append((int(r[ci["Warp Stall Sampling (All Samples)"]] or 0), r[ci["Source"]].strip()))
        except Exception:
            pass
    tot = sum(d[0] for d in data) or 1
    agg = collections.Counter()
    for s, t in data:
        agg[t.split()[0] if t else "?"] += s
    print("stall samples by opcode:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in agg.most_common(top)))

if __name__ == "__main__":
    raw(sys.argv[1])
    source(sys.argv[1])
