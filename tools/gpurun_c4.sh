# c4 strong-shard line (64-query fixed set) on the z-plane marches + a per-kernel launch list at 255^3
ncu --nvtx --nvtx-include "solve/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/c4_launches.csv python tools/prof_3d.py --m 255 --n 60 --random-basis --iters 2 --prof-only > gpurun_out/c4_launch.log 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/c4_launches.csv")) if len(r) > 10]
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value"); ui = hdr.index("Metric Unit")
t = collections.defaultdict(list)
for r in rows[1:]:
    v = float(r[vi].replace(",", "")); v = v / 1e3 if r[ui] == "nsecond" else (v * 1e3 if r[ui] == "msecond" else v)
    t[r[ki].split("(")[0]].append(v)
for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:45s} n={len(v):3d} mean_us={sum(v)/len(v):9.1f}")
PY
timeout 1800 python bench.py --config c4 --queries 64 --steps 1 --warmup 1 > gpurun_out/c4_bench.json 2> gpurun_out/c4_bench.err
tail -1 gpurun_out/c4_bench.json | cut -c1-400
