"""Top SASS instructions by warp-stall samples from `ncu --page source --csv`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
si = hdr.index("Warp Stall Sampling (All Samples)")
ei = hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
body = [r for r in rows[2:] if len(r) == len(hdr)]
tot = sum(float(r[si] or 0) for r in body)
print("total samples", tot)
for k, r in sorted(enumerate(body), key=lambda kr: -float(kr[1][si] or 0))[:n]:
    st = sorted(((float(r[i] or 0), hdr[i]) for i in stall_cols), reverse=True)[:3]
    print(f"{k:5d} {float(r[si]) / tot * 100:5.1f}% exec={r[ei]:>8} {r[1].strip()[:60]:60s} " +
          " ".join(f"{h[6:]}={v:.0f}" for v, h in st if v > 0))
