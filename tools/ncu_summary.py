"""Summarise an ncu report (per kernel: time, DRAM bytes, throughput, DMMA, stalls).

usage: python tools/ncu_summary.py REPORT.ncu-rep [alg_bytes_json] > profiles/X.md
"""
import csv
import io
import json
import subprocess
import sys

M = {
    "time_us": "gpu__time_duration.sum",
    "dram_rd_MB": "dram__bytes_read.sum",
    "dram_wr_MB": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "dmma_pct": "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "fp64_pct": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
}


def main():
    rep = sys.argv[1]
    raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                  stderr=subprocess.DEVNULL).decode()
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {k: (hdr.index(v) if v in hdr else None) for k, v in M.items()}
    stall = [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled")]

    def f(r, i):
        try:
            return float(r[i])
        except Exception:
            return float("nan")

    print(f"# ncu summary: `{rep}`\n")
    print("units: " + ", ".join(f"{k}={units[i]}" for k, i in col.items() if i is not None) + "\n")
    print("| kernel | " + " | ".join(M) + " | top stalls |")
    print("|---" * (len(M) + 2) + "|")
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0]
        vals = [f"{f(r, i):.4g}" if i is not None else "NA" for i in col.values()]
        st = sorted(((f(r, i), hdr[i].replace("smsp__average_warps_issue_stalled_", "")
                      .replace("_per_issue_active.ratio", "")) for i in stall), reverse=True)[:3]
        print(f"| {name} | " + " | ".join(vals) + " | " +
              ", ".join(f"{n} {v:.1f}" for v, n in st) + " |")


if __name__ == "__main__":
    main()
