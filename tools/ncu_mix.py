"""Executed-instruction mix of one kernel (ncu source page): python tools/ncu_mix.py REP REGEX"""
import csv, io, subprocess, sys, collections
raw = subprocess.check_output(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "-k", "regex:" + sys.argv[2],
                               "--launch-count", "1"], stderr=subprocess.DEVNULL).decode()
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ie = hdr.index("Instructions Executed")
seen, mix, tot = set(), collections.Counter(), 0
for r in rows[2:]:
    if len(r) < len(hdr) or not r[ie].isdigit():
        continue
    if r[0] in seen:
        break
    seen.add(r[0])
    n = int(r[ie]); tot += n
    ins = r[1].strip().split()
    op = ins[1] if ins and ins[0].startswith("@") else (ins[0] if ins else "?")
    mix[op.split(".")[0]] += n
print("total", tot)
for op, n in mix.most_common(25):
    print(f"{op:12s} {n/1e6:8.2f}M {100*n/tot:5.1f}%")
