"""Per-source-line warp-stall samples from an ncu report (source page, cuda+sass).

    python tools/ncu_lines.py <report.ncu-rep> [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], "?", None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit() and r[2] == "-":
        d = dict(zip(hdr[4:], r[4:]))
        rows.append((int(d.get("Warp Stall Sampling (All Samples)", 0) or 0), fname, int(r[0]), r[1][:90],
                     int(d.get("Instructions Executed", 0) or 0)))
tot = sum(x[0] for x in rows) or 1
rows.sort(reverse=True)
print(f"total samples {tot}")
for s, f, ln, src, ex in rows[:top]:
    print(f"{100*s/tot:5.1f}% {f}:{ln:<4} inst={ex:<11} {src}")
