"""Key issue/memory metrics per kernel of an ncu report: python tools/ncu_brief.py REP [regex]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
args = ["ncu", "-i", rep, "--page", "raw", "--csv"] + (["-k", "regex:" + sys.argv[2]] if len(sys.argv) > 2 else [])
rows = list(csv.reader(io.StringIO(subprocess.check_output(args, stderr=subprocess.DEVNULL).decode())))
hdr = rows[0]
K = [("time_us", "gpu__time_duration.sum"), ("inst_M", "smsp__inst_executed.sum"),
     ("issue%", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
     ("dram_rd_MB", "dram__bytes_read.sum"), ("dram_wr_MB", "dram__bytes_write.sum"),
     ("dram%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
     ("dmma%", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
     ("fp64%", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
     ("st_wait", "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"),
     ("st_bar", "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio"),
     ("st_lsb", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"),
     ("st_ssb", "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio"),
     ("st_mio", "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio"),
     ("st_math", "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"),
     ("bank_conf", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")]
idx = {k: hdr.index(m) for k, m in K if m in hdr}
print("kernel".ljust(28) + "".join(k.rjust(11) for k, _ in K if k in idx))
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")][:27]
    vals = []
    for k, _ in K:
        if k not in idx:
            continue
        v = r[idx[k]]
        try:
            f = float(v)
            if k == "inst_M":
                f /= 1e6
            vals.append(f"{f:11.2f}")
        except ValueError:
            vals.append(v[:11].rjust(11))
    print(name.ljust(28) + "".join(vals))
