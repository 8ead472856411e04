"""Per-CUDA-line stall samples and executed instructions of an ncu report (analysis aid).
usage: python scripts/ncu_lines.py REPORT.ncu-rep [top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, out = None, []
for r in csv.reader(io.StringIO(txt)):
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if not r or r[0] == "Line No" or len(r) < 8 or r[2] != "-":
        continue
    try:
        st, ins = int(r[4]), int(r[7])
    except ValueError:
        continue
    out.append((st, ins, cur, r[0], r[1].strip()[:100]))
tot = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
print(f"stall samples {tot}, instructions {ti}")
for o in sorted(out, reverse=True)[:top]:
    print(f"{100 * o[0] / tot:5.1f}% {100 * o[1] / ti:5.1f}% {o[2]}:{o[3]} {o[4]}")
