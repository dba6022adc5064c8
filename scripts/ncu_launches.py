"""Per-launch device times from an `ncu --metrics gpu__time_duration.sum --csv --log-file` capture:
writes a compact CSV and prints each kernel's share of the captured time."""
import csv
import sys
from collections import defaultdict

src, dst = sys.argv[1], sys.argv[2]
lines = [ln for ln in open(src) if not ln.startswith("==")]
rows = list(csv.reader(lines))
h = rows[0]
out = []
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") == "gpu__time_duration.sum":
        name = d["Kernel Name"].split("(")[0].replace("unnamed>::", "").replace("lbk::", "")
        out.append((d["ID"], name, d["Grid Size"], d["Block Size"], float(d["Metric Value"])))
with open(dst, "w") as fh:
    fh.write("id,kernel,grid,block,gpu_time_ns\n")
    for o in out:
        fh.write(f'{o[0]},"{o[1]}","{o[2]}","{o[3]}",{o[4]:.0f}\n')
agg = defaultdict(float)
for o in out:
    agg[o[1].split("<")[0]] += o[4]
tot = sum(agg.values())
print({k: round(v / tot, 4) for k, v in agg.items()}, "launches", len(out))
