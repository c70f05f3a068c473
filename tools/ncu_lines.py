"""Per-CUDA-source-line instructions executed and stall samples of one kernel in an ncu
report: python tools/ncu_lines.py REP KERNEL_REGEX [N]"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                               "-k", "regex:" + kre, "--launch-count", "1"], stderr=subprocess.DEVNULL).decode()
rows = list(csv.reader(io.StringIO(raw)))
cur, hdr = None, None
inst, samp, src = collections.Counter(), collections.Counter(), {}
stalls = collections.defaultdict(collections.Counter)
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 8:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    k = (cur, ln)
    def fv(name):
        try:
            return float(r[hdr.index(name)])
        except (ValueError, IndexError):
            return 0.0
    inst[k] += fv("Instructions Executed")
    samp[k] += fv("Warp Stall Sampling (All Samples)")
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                stalls[k][h[6:]] += float(r[i] or 0)
            except ValueError:
                pass
    src[k] = r[1][:80]
ti, ts = sum(inst.values()) or 1, sum(samp.values()) or 1
print(f"total inst {ti:.0f} samples {ts:.0f}")
for k, v in samp.most_common(top):
    st = ", ".join(f"{n} {x:.0f}" for n, x in stalls[k].most_common(3))
    print(f"{100*v/ts:5.1f}% samp {100*inst[k]/ti:5.1f}% inst {k[0]}:{k[1]} {src[k]} [{st}]")
