"""Hottest SASS instructions of an ncu source page (--page source --csv --print-source sass).
usage: python scripts/ncu_hot.py src.csv [top] [addr_lo addr_hi]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ia, isrc, isamp = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
iex = hdr.index("Instructions Executed")
stalls = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[isamp] or 0) for r in data)
print(f"total samples {tot:.0f}")
rng = None
if len(sys.argv) > 4:
    rng = (int(sys.argv[3], 16), int(sys.argv[4], 16))
sel = [r for r in data if rng is None or rng[0] <= int(r[ia], 16) <= rng[1]]
if rng:
    for r in sel:
        st = sorted(((float(r[i] or 0), hdr[i][6:]) for i in stalls), reverse=True)[:3]
        print(f"{r[ia]} {float(r[isamp] or 0):6.0f} {r[iex]:>8s} {r[isrc][:60]:60s} " + " ".join(f"{n}={v:.0f}" for v, n in st if v))
else:
    for r in sorted(sel, key=lambda r: -float(r[isamp] or 0))[:top]:
        st = sorted(((float(r[i] or 0), hdr[i][6:]) for i in stalls), reverse=True)[:3]
        print(f"{r[ia]} {float(r[isamp] or 0):6.0f} {r[iex]:>8s} {r[isrc][:60]:60s} " + " ".join(f"{n}={v:.0f}" for v, n in st if v))
    agg = {}
    for r in data:
        for i in stalls:
            agg[hdr[i][6:]] = agg.get(hdr[i][6:], 0) + float(r[i] or 0)
    print(sorted(((round(v), k) for k, v in agg.items()), reverse=True)[:12])
