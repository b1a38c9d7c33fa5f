"""Per-source-line share of warp-stall samples and executed instructions from
an ncu report: python tools/ncu_lines.py REPORT.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, out = None, None, []
for r in csv.reader(io.StringIO(txt)):
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 10 or r[2] != "-":
        continue
    try:
        samp, inst = int(r[4]), int(r[7])
    except ValueError:
        continue
    out.append((samp, inst, cur, r[0], r[1][:100]))
tot = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
print("total samples", tot, "warp instructions", ti)
for o in sorted(out, reverse=True)[:top]:
    print(f"{o[0] / tot * 100:5.1f}% {o[1] / ti * 100:5.1f}%i {o[2]}:{o[3]} {o[4]}")
