"""Summarise an ncu --set full report: key throughput, traffic and stall metrics."""
import csv
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
    "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "local_load", "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum",
]


def main(path, sites=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for v in rows[2:]:
        print("kernel:", v[h.index("Kernel Name")][:80])
        d = dict(zip(h, v))
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k]:>16s} {units[h.index(k)]}")
        stalls = {k: float(d[k]) for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio") and d[k] not in ("", "n/a")}
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:8]
        print("  top stalls (warps per issue):", ", ".join(f"{k.split('stalled_')[1].split('_per')[0]}={v:.2f}" for k, v in top))
        if sites:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rb = float(d["dram__bytes_read.sum"].replace(",", "")) * scale[units[h.index("dram__bytes_read.sum")]]
            wb = float(d["dram__bytes_write.sum"].replace(",", "")) * scale[units[h.index("dram__bytes_write.sum")]]
            print(f"  dram bytes/site: read {rb/sites:.1f} write {wb/sites:.1f}  (algorithmic 304 + 304)")
            print(f"  dram bytes/launch: {rb + wb:.6e}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None)
