# session-4 round-2 end check on HEAD: smoke, c2 bench line (driver-equivalent), launch list, full GPU suite
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s4_smoke.log 2>&1; tail -1 gpurun_out/s4_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/s4_bench.json 2> gpurun_out/s4_bench.err
tail -1 gpurun_out/s4_bench.json | cut -c1-300
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/s4_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --streams 1 \
    > gpurun_out/s4_launches.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s4_gpu_tests.log 2>&1; tail -2 gpurun_out/s4_gpu_tests.log
