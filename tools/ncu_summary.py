"""Summarise an ncu --set full report of the select path into profiles/ JSON.

    python tools/ncu_summary.py gpurun_out/prof_r01.ncu-rep profiles/ncu_select_r01.json "<capture note>"

Keeps the metrics DESIGN.md and bench.py cite (dram bytes in MB per launch,
duration in us, occupancy, stall samples), averaged over the captured launches
of each kernel.
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEEP = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
    "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.avg.per_cycle_active", "smsp__inst_executed.sum",
    "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_barrier",
    "smsp__pcsamp_warps_issue_stalled_short_scoreboard", "smsp__pcsamp_warps_issue_stalled_wait",
    "smsp__pcsamp_warps_issue_stalled_lg_throttle", "smsp__pcsamp_warps_issue_stalled_membar",
    "smsp__pcsamp_warps_issue_stalled_drain", "smsp__pcsamp_warps_issue_stalled_mio_throttle",
    "smsp__pcsamp_warps_issue_stalled_no_instructions", "smsp__pcsamp_warps_issue_stalled_selected",
    "smsp__pcsamp_warps_issue_stalled_not_selected", "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
    "smsp__pcsamp_warps_issue_stalled_dispatch_stall", "smsp__pcsamp_warps_issue_stalled_branch_resolving",
    "smsp__pcsamp_sample_count",
    "lts__t_sectors_srcunit_tex_op_write.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
]
SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3,  # -> MB
         "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}  # -> us


def main():
    rep, out, note = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    acc = defaultdict(lambda: defaultdict(list))
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        for m in KEEP:
            if m not in col:
                continue
            v = r[col[m]].replace(",", "")
            try:
                x = float(v) * SCALE.get(units[col[m]], 1.0)
            except ValueError:
                continue
            acc[name][m].append(x)
    res = {"capture": note, "units": "MB for bytes, us for durations", "kernels": {}}
    for name, ms in acc.items():
        res["kernels"][name] = {m: sum(v) / len(v) for m, v in ms.items()}
        res["kernels"][name]["launches"] = max(len(v) for v in ms.values())
    sel = [k for k in res["kernels"] if "stream_kernel" in k]
    if sel:
        s = res["kernels"][sel[0]]
        res["dram_bytes_per_launch"] = (s.get("dram__bytes_read.sum", 0) + s.get("dram__bytes_write.sum", 0)) * 1e6
    json.dump(res, open(out, "w"), indent=1, sort_keys=True)
    print(json.dumps(res, indent=1, sort_keys=True)[:3000])


if __name__ == "__main__":
    main()
