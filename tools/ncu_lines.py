"""Per-CUDA-source-line warp-stall samples (or executed instructions) of one
kernel from an ncu report:
python tools/ncu_lines.py report.ncu-rep kernel_regex [top] [inst]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
# column 4: warp-stall samples; 7: instructions executed ("inst")
col = 7 if len(sys.argv) > 4 and sys.argv[4] == "inst" else 4
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv",
                      "--print-source", "cuda,sass", "--kernel-name",
                      "regex:" + kern, "-c", "1"],
                     capture_output=True, text=True).stdout
fname = ""
rows = []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No" or r[0] == "Function Name":
        continue
    if r[0] and r[0] != "":
        try:
            s = float(r[col])
        except (ValueError, IndexError):
            continue
        rows.append((s, f"{fname}:{r[0]}", r[1].strip()[:100]))
tot = sum(x[0] for x in rows) or 1
for s, loc, src in sorted(rows, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}% {loc:18s} {src}")
