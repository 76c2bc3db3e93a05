"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) by kernel."""
import collections, csv, re, sys

def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hi]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    gi = hdr.index("Grid Size") if "Grid Size" in hdr else None
    out = []
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = re.sub(r"\(.*", "", r[ki])
        m = re.search(r"(gemm_kernel|gemm_grouped_kernel)<(\d+), (\d+)", r[ki])
        if m:
            name = f"{m.group(1)}<{m.group(2)},{m.group(3)}>"
        name = name.replace("pevd::<unnamed>::", "").replace("void ", "")
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(u, 1e-6)
        out.append((name, v * scale, r[gi] if gi is not None else ""))
    return out

if __name__ == "__main__":
    recs = load(sys.argv[1])
    tot, cnt = collections.Counter(), collections.Counter()
    for name, ms, _ in recs:
        tot[name] += ms
        cnt[name] += 1
    T = sum(tot.values())
    print(f"{'ms':>10} {'share':>6} {'launches':>8}  kernel")
    for k, v in tot.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
        print(f"{v:10.2f} {100 * v / T:5.1f}% {cnt[k]:8d}  {k}")
    print(f"{T:10.2f} total ms over {len(recs)} launches")
