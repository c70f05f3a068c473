# 2D K3 split experiment (prolongation pass + sweep march) at c2, plus the order A/B of the c2 bench
python tools/prof_c2.py --build /tmp/c2basis.pt > /dev/null 2>&1
for V in 0 262144; do
  echo "v2off=$V: $(RBS_DISABLE_V2=$V PROF_GRAPH=1 python tools/prof_c2.py --load /tmp/c2basis.pt --iters 20 | tr '\n' ' ')"
done
RBS_DISABLE_V2=262144 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c1 or c2 or ragged" > gpurun_out/s3_tests.log 2>&1; tail -1 gpurun_out/s3_tests.log
timeout 900 python -m pytest tests/test_gpu_zmarch.py -x -q > gpurun_out/s3_ztests.log 2>&1; tail -1 gpurun_out/s3_ztests.log
python bench.py --steps 16 --warmup 4 --no-cpu-baseline --order given > gpurun_out/s3_bench_given.json 2>/dev/null
python bench.py --steps 16 --warmup 4 --no-cpu-baseline --order contrast > gpurun_out/s3_bench_contrast.json 2>/dev/null
for f in given contrast; do python -c "
import json; d=json.loads(open('gpurun_out/s3_bench_$f.json').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), d['clocks']['sm_mhz'], d['config']['its_min_med_max'])"; done
python bench.py --config case1 --steps 6 --warmup 3 > gpurun_out/s3_case1.json 2>/dev/null; tail -1 gpurun_out/s3_case1.json | cut -c1-200
