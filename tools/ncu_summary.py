"""Key metrics of every kernel in an ncu report (ncu -i ... --page raw --csv)."""
import csv
import io
import subprocess
import sys

WANT = [
    ("launch__grid_size", "grid"), ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("lts__t_bytes.sum", "l2_bytes"), ("lts__t_sector_hit_rate.pct", "l2_hit%"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit%"), ("l1tex__t_bytes.sum", "l1_bytes"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy%"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall_long_sb"),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "stall_lg_thr"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall_wait"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall_math"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall_short_sb"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall_barrier"),
    ("smsp__inst_executed.sum", "inst"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "ld_req"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "ld_sectors"),
]


def summary(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")][:70]
        out.append(name)
        for m, short in WANT:
            if m in hdr:
                i = hdr.index(m)
                out.append(f"  {short:16s} {vals[i]} {units[i]}")
    return "\n".join(out)


if __name__ == "__main__":
    for r in sys.argv[1:]:
        print(summary(r))
