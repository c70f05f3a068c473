"""Top SASS hot spots of an ncu report (source page): python tools/ncu_hot.py REP [N] [kernel-regex]"""
import csv, io, re, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
args = ["ncu", "-i", rep, "--page", "source", "--csv"]
if len(sys.argv) > 3:
    args += ["-k", "regex:" + sys.argv[3]]
raw = subprocess.check_output(args, stderr=subprocess.DEVNULL).decode()
lines = raw.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(l for l in lines if not l.startswith('"Kernel Name"')))))
hdr = rows[0]
si = hdr.index("Warp Stall Sampling (All Samples)")
st = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[si] or 0) for r in rows[1:] if len(r) > si and r[si].replace('.', '', 1).isdigit())
agg = {}
out = []
for r in rows[1:]:
    if len(r) <= si or not r[si].replace('.', '', 1).isdigit():
        continue
    v = float(r[si]); op = r[1].strip().split()[0] if r[1].strip() else "?"
    if op.startswith("@"):
        op = r[1].strip().split()[1]
    op = op.split(".")[0]
    agg[op] = agg.get(op, 0) + v
    reasons = sorted(((float(r[i] or 0), hdr[i][6:]) for i in st), reverse=True)[:2]
    out.append((v, r[0][-5:], r[1].strip()[:60], reasons))
print(f"total samples {tot:.0f}")
print("by opcode:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:14]))
for v, a, s, rs in sorted(out, reverse=True)[:top]:
    print(f"{100*v/tot:5.1f}% {a} {s:60s} " + " ".join(f"{n}={x:.0f}" for x, n in rs))
