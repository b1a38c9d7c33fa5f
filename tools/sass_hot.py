"""Hot SASS of an ncu source-page export (tools/ncu_capture.sh *_sass.csv):
instructions sorted by address with executed warp-instruction counts,
printing only the blocks that execute at least FRAC of the total.
python tools/sass_hot.py FILE [frac]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.002
hdr = next(r for r in rows if r and r[0] == "Address")
ie = hdr.index("Instructions Executed")
sa = hdr.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows if r and r[0].startswith("0x")]
tot = sum(int(r[ie] or 0) for r in body)
print("total warp instructions", tot)
for r in body:
    c = int(r[ie] or 0)
    if c >= frac * tot:
        print(f"{r[0][-5:]} {c / tot * 100:6.2f}% samp {r[sa]:>6} {r[1].strip()}")
