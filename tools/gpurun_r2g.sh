# z-march residual-projection of the symmetric preconditioner (k_xrz<RES> + k_wtr): parity, then
# A/B per pass at 255^3 (B = 8, n = 40: c5's batch and basis width; B = 16, n = 60: c4's)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_zmarch.py tests/test_gpu_next3.py -q > gpurun_out/g_tests.log 2>&1; tail -2 gpurun_out/g_tests.log
for cfg in "--B 8 --n 40" "--B 16 --n 60"; do
  echo "== $cfg new";  timeout 600 python tools/prof_3d.py --m 255 $cfg --random-basis --iters 3 --precond 1 2>&1 | tail -1
  echo "== $cfg flat"; RBS_DISABLE_V2=524288 timeout 600 python tools/prof_3d.py --m 255 $cfg --random-basis --iters 3 --precond 1 2>&1 | tail -1
done > gpurun_out/g_ab.txt
cat gpurun_out/g_ab.txt
