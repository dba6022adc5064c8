"""Per-launch DRAM bytes per site and time from an ncu --metrics --csv log."""
import csv
import sys

rows = [r for r in csv.reader(ln for ln in open(sys.argv[1]) if not ln.startswith("=="))]
sites = float(sys.argv[2])
h, data = rows[0], {}
for r in rows[1:]:
    d = dict(zip(h, r))
    k = (int(d["ID"]), d["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", ""))
    data.setdefault(k, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
for (i, name), m in sorted(data.items()):
    print(f"  {i:2d} {name:34s} t={m['gpu__time_duration.sum'] / 1e3:8.1f} us  read/site={m['dram__bytes_read.sum'] / sites:6.1f}"
          f"  write/site={m['dram__bytes_write.sum'] / sites:6.1f}")
