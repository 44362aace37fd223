"""Hottest SASS instructions of a kernel from `ncu -i REP --page source --csv` output.

    ncu -i rep --page source --csv > src.csv; python tools/ncu_hot.py src.csv [kernel-substring] [N]
"""
import csv
import io
import sys

path = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
text = open(path).read()
blocks = text.split('"Kernel Name",')[1:]
for b in blocks:
    name, rest = b.split("\n", 1)
    if want not in name:
        continue
    rows = list(csv.DictReader(io.StringIO(rest)))
    tot = sum(float(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
    print(name.strip(), f"total samples {tot:.0f}")
    stall_cols = [c for c in rows[0] if c.startswith("stall_") and "Not Issued" not in c]
    agg = {c: sum(float(r[c] or 0) for r in rows) for c in stall_cols}
    print("  by reason:", ", ".join(f"{c[6:]} {100 * v / tot:.1f}%" for c, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]))
    rows.sort(key=lambda r: -float(r["Warp Stall Sampling (All Samples)"] or 0))
    for r in rows[:top]:
        s = float(r["Warp Stall Sampling (All Samples)"] or 0)
        st = sorted(((float(r[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
        print(f"  {100 * s / tot:5.2f}% {r['Address']:>6} {r['Source'][:60]:60s} " + " ".join(f"{n}:{v:.0f}" for v, n in st if v > 0))
