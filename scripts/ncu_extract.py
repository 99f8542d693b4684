"""Pull the metrics that matter out of `ncu --set full` reports into one JSON file.
Usage: python scripts/ncu_extract.py out.json name=report.ncu-rep [name=report.ncu-rep ...]"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_rate_pct",
    "lts__t_sectors.sum": "l2_sectors",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "smsp__cycles_active.avg": "smsp_cycles_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_slots_busy_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__shared_mem_per_block_dynamic": "dynamic_smem_per_block",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct": "global_load_sector_efficiency_pct",
}
STALL = "smsp__average_warps_issue_stalled_"


def scale(v, unit):
    mult = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9,
            "second": 1.0, "us": 1e-6, "ms": 1e-3, "ns": 1e-9}
    return v * mult.get(unit, 1.0)


out = {}
for arg in sys.argv[2:]:
    name, path = arg.split("=", 1)
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    launches = []
    for vals in rows[2:]:
        rec, stalls = {}, {}
        for h, u, v in zip(hdr, units, vals):
            if h == "Kernel Name":
                rec["kernel"] = v.split("(")[0]
            if h in KEYS and v not in ("", "n/a"):
                try:
                    rec[KEYS[h]] = scale(float(v.replace(",", "")), u)
                except ValueError:
                    pass
            if h.startswith(STALL) and h.endswith("_per_issue_active.ratio") and "not_issued" not in h:
                try:
                    stalls[h[len(STALL):-len("_per_issue_active.ratio")]] = round(float(v), 3)
                except ValueError:
                    pass
        rec["stall_per_issue_top"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
        if "dram_read" in rec and "dram_write" in rec:
            rec["dram_bytes"] = rec["dram_read"] + rec["dram_write"]
        launches.append(rec)
    out[name] = launches
json.dump(out, open(sys.argv[1], "w"), indent=1)
for k, v in out.items():
    for r in v:
        print(k, {q: r.get(q) for q in ("kernel", "duration", "dram_bytes", "dram_throughput_pct", "fp64_pipe_pct", "issue_slots_busy_pct", "l2_hit_rate_pct", "achieved_occupancy_pct", "registers_per_thread")}, r["stall_per_issue_top"])
