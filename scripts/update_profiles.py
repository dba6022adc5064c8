"""Refresh profiles/ from the artefacts scripts/gpu_full.sh leaves in gpurun_out/:
ncu summary + SASS stall regions of the step kernel, the launch list, traffic.json
(keyed to the current source hash) and the bench lines.

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
rep = os.path.join(G, "prof_kstep_c5.ncu-rep")
sites = 512 * 512 * 64
summ = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), rep, str(sites)],
                      capture_output=True, text=True, check=True).stdout
sass_csv = os.path.join(G, "kstep_sass.csv")
with open(sass_csv, "w") as fh:
    subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], stdout=fh, check=True)
regions = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_sass_regions.py"), sass_csv],
                         capture_output=True, text=True, check=True).stdout
with open(os.path.join(P, f"{tag}_ncu_full_kstep_c5.txt"), "w") as fh:
    fh.write(summ + regions)
launches = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_launches.py"),
                           os.path.join(G, "launches.csv"), os.path.join(P, f"{tag}_ncu_launches_c5.csv")],
                          capture_output=True, text=True, check=True).stdout
print("launch shares:", launches.strip())
vals = {}
for ln in summ.splitlines():
    parts = ln.split()
    if len(parts) >= 2 and parts[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        vals[parts[0]] = float(parts[1]) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[parts[2]]
tr = {"k_step@c5": {
    "dram_bytes_per_launch": vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"],
    "dram_read_bytes_per_site": round(vals["dram__bytes_read.sum"] / sites, 1),
    "dram_write_bytes_per_site": round(vals["dram__bytes_write.sum"] / sites, 1),
    "src_hash": bench.src_hash(),
    "source": f"profiles/{tag}_ncu_full_kstep_c5.txt (ncu --set full, 512x512x64, 1 launch)"}}
with open(os.path.join(P, "traffic.json"), "w") as fh:
    json.dump(tr, fh, indent=1)
print("traffic:", tr)
for f in ("default", "c3", "c2", "ref", "mrt", "ch"):
    src = os.path.join(G, f"bench_{f}.json")
    if os.path.exists(src) and os.path.getsize(src) > 0:
        shutil.copy(src, os.path.join(P, f"{tag}_bench_{f}.json"))
