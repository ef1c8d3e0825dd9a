"""Summarise an `ncu --page source --csv --print-source sass` dump: top SASS lines by warp-stall samples."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iall, inot = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), \
    hdr.index("Warp Stall Sampling (Not-issued Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[iall] or 0), int(r[inot] or 0), r[ia], r[isrc]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
print("total samples", tot)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for a, b, addr, src in sorted(data, reverse=True)[:n]:
    print(f"{a:7d} {100.0 * a / tot:5.1f}% {b:7d} {addr} {src[:90]}")
