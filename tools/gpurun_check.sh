# head check: smoke, GPU suite, c2 bench line
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/chk_smoke.log 2>&1; tail -1 gpurun_out/chk_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/chk_gpu_tests.log 2>&1; tail -2 gpurun_out/chk_gpu_tests.log
python bench.py --steps 20 --warmup 5 > gpurun_out/chk_bench.json 2> gpurun_out/chk_bench.err
tail -1 gpurun_out/chk_bench.json | cut -c1-400
