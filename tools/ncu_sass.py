"""Per-instruction executed counts of one kernel in an ncu report (SASS order).
usage: python tools/ncu_sass.py REP KERNEL_REGEX [min_pct]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
minp = float(sys.argv[3]) if len(sys.argv) > 3 else 0.3
raw = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre,
                               "--launch-count", "1"], stderr=subprocess.DEVNULL).decode()
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ie, si = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
lines = []
for r in rows[2:]:
    if len(r) < len(hdr) or not r[ie].isdigit():
        continue
    lines.append((r[0][-5:], r[1].strip(), int(r[ie]), float(r[si] or 0)))
tot = sum(l[2] for l in lines)
ts = sum(l[3] for l in lines) or 1
print(f"total warp-instructions {tot}")
for a, s, n, st in lines:
    if 100 * n / tot >= minp or 100 * st / ts >= minp:
        print(f"{a} {100*n/tot:5.2f}% st{100*st/ts:5.2f}% {s[:80]}")
