"""Top stalled SASS instructions of one captured launch (needs -lineinfo and --import-source at capture):
    python tools/ncu_hot.py <report.ncu-rep> <launch index> [top=25]"""
import csv
import io
import subprocess
import sys

rep, idx = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(idx), "--launch-count", "1",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
si = h.index("Warp Stall Sampling (All Samples)")
src = h.index("Source")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(r[si] or 0) for r in rows[1:] if len(r) > si)
print(lines[0][:160])
print(f"total samples {tot:.0f}")
ranked = sorted(rows[1:], key=lambda r: -float(r[si] or 0) if len(r) > si else 0)[:top]
for r in ranked:
    st = sorted(((float(r[i] or 0), h[i][6:]) for i in stall_cols), reverse=True)[:3]
    print(f"{float(r[si]) / tot * 100:5.1f}%  {r[src].strip()[:60]:60s} " + ", ".join(f"{n} {v:.0f}" for v, n in st if v))
