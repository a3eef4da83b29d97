"""Top stall-sampled SASS lines of an ncu --page source --csv --print-source sass export.
usage: python tools/ncu_hot.py export.csv [N] — prints the N hottest instructions (in program
order) with their share of all warp samples and of the not-issued samples."""
import csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
isrc, iall, ino = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), \
    hdr.index("Warp Stall Sampling (Not-issued Samples)")
body = [r for r in rows[2:] if len(r) == len(hdr)]
tot = sum(int(r[iall] or 0) for r in body)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print("total samples", tot)
idx = sorted(range(len(body)), key=lambda i: -int(body[i][iall] or 0))[:n]
for i in sorted(idx):
    r = body[i]
    print(f"{i:5d} {int(r[iall]) / tot * 100:5.1f}% {int(r[ino]) / tot * 100:5.1f}%  {r[isrc].strip()[:90]}")
