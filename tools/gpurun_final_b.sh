# final round-2 measurements, part B: the GPU test suite, smoke, sanitizers
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/final_gpu_tests.log 2>&1; tail -2 gpurun_out/final_gpu_tests.log
for t in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 1 python tools/sanitize.py > gpurun_out/final_$t.log 2>&1
  echo "$t rc=$?"; tail -2 gpurun_out/final_$t.log
done
