# final-build check: smoke, the whole GPU suite, the driver-equivalent c2 line, c4 stand-alone RBI (16 queries)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/j_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/j_gpu_tests.log 2>&1; tail -2 gpurun_out/j_gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/j_c2.json 2> gpurun_out/j_c2.err
echo "c2 rc=$?"; tail -1 gpurun_out/j_c2.json | cut -c1-200
timeout 1500 python bench.py --config c4 --method rbi --queries 16 --steps 1 --warmup 1 > gpurun_out/j_c4_rbi.json 2> gpurun_out/j_c4_rbi.err
echo "c4 rbi rc=$?"; tail -1 gpurun_out/j_c4_rbi.json | cut -c1-300
