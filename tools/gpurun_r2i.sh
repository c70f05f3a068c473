# RBI 3D residual-projection by k_xrz<RES> + k_wtr: parity, then A/B at 255^3 (B = 16, n = 60)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_zmarch.py -q > gpurun_out/i_tests.log 2>&1; tail -2 gpurun_out/i_tests.log
for cfg in "--B 16 --n 60" "--B 8 --n 40"; do
  echo "== $cfg new";  timeout 600 python tools/prof_3d.py --m 255 $cfg --random-basis --iters 3 --rbi 2>&1 | tail -1
  echo "== $cfg flat"; RBS_DISABLE_V2=524288 timeout 600 python tools/prof_3d.py --m 255 $cfg --random-basis --iters 3 --rbi 2>&1 | tail -1
done > gpurun_out/i_ab.txt
cat gpurun_out/i_ab.txt
