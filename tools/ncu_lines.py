"""Per-CUDA-source-line warp-stall samples of one kernel from an ncu report
(ncu --page source --print-source cuda,sass): the lines where the warps wait.
Usage: python tools/ncu_lines.py gpurun_out/prof_score.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, rows, hdr = "?", [], None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    try:
        s_all, s_ni, ins = int(r[4]), int(r[5]), int(r[7])
    except (ValueError, IndexError):
        continue
    rows.append((s_all, s_ni, ins, f"{fname}:{r[0]}", r[1].strip()[:90]))
tot = sum(x[0] for x in rows) or 1
rows.sort(reverse=True)
print(f"total stall samples {tot}")
print(" samples   %all  not-issued  instr-exec  line  source")
for s_all, s_ni, ins, loc, src in rows[:top]:
    print(f"{s_all:8d} {100 * s_all / tot:5.1f}% {s_ni:10d} {ins:11d}  {loc:28s} {src}")
