"""Refresh profiles/ from the artefacts scripts/gpu_final_{a,b,c}.sh
leave in gpurun_out/: ncu summary + per-line stall/instruction shares of the step
kernels, the launch lists, traffic.json (keyed to the current source hash) and
the bench lines.

  python scripts/update_profiles.py [round-tag, default r1]
"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
UNITS = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
traffic_path = os.path.join(P, "traffic.json")
traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}

# (ncu report, launch list, profile suffix, traffic key, sites, lattice)
C5, C3 = 512 * 512 * 64, 128 ** 3
CAPTURES = [("prof_kstep_c5", "launches.csv", "c5", "k_step@c5", C5, "512x512x64"),
            ("prof_kstep_c3", "launches_c3.csv", "c3", "k_step@c3", C3, "128^3"),
            ("prof_kstep_lc", "launches_lc.csv", "lc", "k_step@c5-lc", C5, "512x512x64"),
            ("prof_kstep_c2", "launches_c2.csv", "c2", "k_step@c2", 64 ** 3, "64^3"),
            ("prof_kstep_c4", "launches_c4.csv", "c4", "k_step@c4", 256 ** 3, "256^3"),
            ("prof_kstep_mrt", "launches_mrt.csv", "mrt", "k_step@c5-mrt", C5, "512x512x64"),
            ("prof_kstep_ch", "launches_ch.csv", "ch", "k_step@c5-ch", C5, "512x512x64")]
for rep_name, launch_csv, suffix, key, sites, lat in CAPTURES:
    rep = os.path.join(G, rep_name + ".ncu-rep")
    if not os.path.exists(rep):
        continue
    summ = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), rep, str(sites)],
                          capture_output=True, text=True, check=True).stdout
    src_csv = os.path.join(G, rep_name + "_src.csv")
    with open(src_csv, "w") as fh:
        subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], stdout=fh,
                       check=True)
    lines = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_lines.py"), src_csv, "30"],
                           capture_output=True, text=True, check=True).stdout
    with open(os.path.join(P, f"{tag}_ncu_full_kstep_{suffix}.txt"), "w") as fh:
        fh.write(summ + "\nper source line (share of stall samples, of warp instructions):\n" + lines)
    lpath = os.path.join(G, launch_csv)
    if os.path.exists(lpath):
        shares = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_launches.py"), lpath,
                                 os.path.join(P, f"{tag}_ncu_launches_{suffix}.csv")],
                                capture_output=True, text=True, check=True).stdout
        print(suffix, "launch shares:", shares.strip())
    vals = {}
    for ln in summ.splitlines():
        parts = ln.split()
        if len(parts) >= 3 and parts[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            vals[parts[0]] = float(parts[1]) * UNITS[parts[2]]
    traffic[key] = {
        "dram_bytes_per_launch": vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"],
        "dram_read_bytes_per_site": round(vals["dram__bytes_read.sum"] / sites, 1),
        "dram_write_bytes_per_site": round(vals["dram__bytes_write.sum"] / sites, 1),
        "src_hash": bench.src_hash(),
        "source": f"profiles/{tag}_ncu_full_kstep_{suffix}.txt (ncu --set full, {lat}, 1 launch)"}
    print("traffic:", key, traffic[key])
# the Cahn-Hilliard kernel: DRAM bytes from a metrics-only capture (scripts/gpu_final_c.sh)
ch_csv = os.path.join(G, "ncu_ch_dram.csv")
if not os.path.exists(os.path.join(G, "prof_kstep_ch.ncu-rep")) and os.path.exists(ch_csv):
    import csv
    rows = [r for r in csv.reader(open(ch_csv)) if len(r) > 5]
    i, v = rows[0].index("Metric Name"), rows[0].index("Metric Value")
    m = {r[i]: float(r[v].replace(",", "")) for r in rows[1:]}
    rd, wr = m["dram__bytes_read.sum"], m["dram__bytes_write.sum"]
    shutil.copy(ch_csv, os.path.join(P, f"{tag}_ncu_kstep_ch_dram.csv"))
    traffic["k_step@c5-ch"] = {
        "dram_bytes_per_launch": rd + wr, "dram_read_bytes_per_site": round(rd / C5, 1),
        "dram_write_bytes_per_site": round(wr / C5, 1), "src_hash": bench.src_hash(),
        "source": f"profiles/{tag}_ncu_kstep_ch_dram.csv (ncu --metrics dram__bytes_*, 512x512x64, 1 launch)"}
    print("traffic:", "k_step@c5-ch", traffic["k_step@c5-ch"])
with open(traffic_path, "w") as fh:
    json.dump(traffic, fh, indent=1)
# bench lines: roofline.traffic from the capture above when it was taken on the
# same sources (bench.py reads traffic.json itself, but the bench runs before the
# capture of the same call)
TKEY = {"default": "k_step@c5", "c3": "k_step@c3", "c2": "k_step@c2", "c4": "k_step@c4", "mrt": "k_step@c5-mrt",
        "ch": "k_step@c5-ch", "lc": "k_step@c5-lc"}
for f in ("default", "c3", "c2", "c4", "c5alt", "ref", "mrt", "ch", "lc"):
    src = os.path.join(G, f"bench_{f}.json")
    if os.path.exists(src) and os.path.getsize(src) > 0:
        dst = os.path.join(P, f"{tag}_bench_{f}.json")
        try:
            line = json.loads(open(src).read().strip().splitlines()[-1])
        except Exception:
            shutil.copy(src, dst)
            continue
        e = traffic.get(TKEY.get(f, ""))
        r = line.get("roofline")
        if r is not None and r.get("traffic") is None and e and e.get("src_hash") == line.get("src_hash"):
            r["traffic"] = e["dram_bytes_per_launch"]
            r["traffic_source"] = e["source"]
        with open(dst, "w") as fh:
            fh.write(json.dumps(line) + "\n")
