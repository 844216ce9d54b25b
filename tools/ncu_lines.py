"""Warp-stall samples aggregated per CUDA source line of one captured launch (needs -lineinfo and
--import-source at capture): python tools/ncu_lines.py <report.ncu-rep> [top=25] [launch=0]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
idx = sys.argv[3] if len(sys.argv) > 3 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--launch-skip", idx,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
agg, fname, line, text = {}, "", None, {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0] != "":  # a CUDA source line
        line = (fname, int(r[0]))
        text[line] = r[1].strip()
        continue
    if line is None or len(r) < 5 or r[4] in ("", "-"):
        continue
    agg[line] = agg.get(line, 0.0) + float(r[4])
tot = sum(agg.values()) or 1.0
print(f"total samples {tot:.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{v / tot * 100:5.1f}%  {k[0]}:{k[1]:<5d} {text.get(k, '')[:100]}")
