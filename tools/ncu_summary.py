"""Summarise one kernel launch of an ncu report into the JSON kept under
profiles/ (dev tool; reads the report with `ncu -i`, no GPU needed).

usage: python tools/ncu_summary.py <report.ncu-rep> <out.json> "<what>" [algorithmic_bytes] [kernel substring]
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__cluster_dim_x",
    "sm__cycles_active.avg",
]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    rep, out, what = sys.argv[1], sys.argv[2], sys.argv[3]
    alg = float(sys.argv[4]) if len(sys.argv) > 4 and float(sys.argv[4]) > 0 else None
    want = sys.argv[5] if len(sys.argv) > 5 else ""
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    head, units = rows[0], rows[1]
    ik = head.index("Kernel Name")
    vals = next(r for r in rows[2:] if want in r[ik])
    got, unit = {}, {}
    for m in METRICS:
        if m in head:
            i = head.index(m)
            got[m], unit[m] = vals[i], units[i]
    got["units"] = unit
    rd = float(got["dram__bytes_read.sum"].replace(",", "")) * SCALE[unit["dram__bytes_read.sum"]]
    wr = float(got["dram__bytes_write.sum"].replace(",", "")) * SCALE[unit["dram__bytes_write.sum"]]
    summary = {"what": what, "kernel": vals[head.index("Kernel Name")] if "Kernel Name" in head else None,
               "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr}
    if alg:
        summary["algorithmic_bytes"] = alg
        summary["traffic_over_algorithmic"] = round((rd + wr) / alg, 3)
    summary["metrics"] = got
    json.dump(summary, open(out, "w"), indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
