"""Summarise ncu captures into profiles/*.md (key counters only)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_eligible.avg.per_cycle_active", "sm__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum",
        "l1tex__t_sector_pipe_lsu_mem_local_op_ld_hit_rate.pct", "sass__inst_executed_local_loads",
        "sass__inst_executed_local_stores", "smsp__inst_executed.sum"]


def summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    lines = []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        lines.append(f"### {name[:80]}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"- `{k}` = {r[i]} {units[i]}")
    return "\n".join(lines)


if __name__ == "__main__":
    rep, title = sys.argv[1], sys.argv[2]
    print(f"# {title}\n\nSource: `{rep}` (`ncu --set full --clock-control none`)\n")
    print(summary(rep))
