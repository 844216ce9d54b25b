"""Compare bench --breakdown logs side by side: python tools/cmp_breakdown.py a.log b.log ..."""
import json
import sys

runs = []
for path in sys.argv[1:]:
    ks, val = {}, None
    for line in open(path):
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        if "kernel" in d:
            ks[d["kernel"]] = d["ms_per_launch"]
        elif "metric" in d:
            val = d["value"]
    runs.append((path, ks, val))
names = sorted({k for _, ks, _ in runs for k in ks}, key=lambda k: -runs[0][1].get(k, 0))
print("%-20s" % "kernel" + "".join("%12s" % p.split("/")[-1][-16:-4] for p, _, _ in runs))
for k in names:
    print("%-20s" % k + "".join("%12.4f" % ks.get(k, float("nan")) for _, ks, _ in runs))
print("%-20s" % "STEP ms" + "".join("%12.4f" % (v or float("nan")) for _, _, v in runs))
