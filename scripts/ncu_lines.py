"""Per-CUDA-source-line totals from `ncu -i REP --page source --csv --print-source cuda,sass`:
warp-level instructions executed and stall samples, top lines first.
  python scripts/ncu_lines.py dump.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, hdr, out = None, None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 2 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0] not in ("",):
        try:
            inst = int(r[hdr.index("Instructions Executed")])
            samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except ValueError:
            continue
        out.append((samp, inst, f"{fname}:{r[0]}", r[1][:70]))
tot_s = sum(o[0] for o in out) or 1
tot_i = sum(o[1] for o in out) or 1
print(f"total samples {tot_s}, warp instructions {tot_i}")
for s, i, loc, src in sorted(out, reverse=True)[:top]:
    print(f"{100*s/tot_s:5.1f}% samp {100*i/tot_i:5.1f}% inst  {loc:24s} {src}")
