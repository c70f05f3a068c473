# compact r (sweep colour only) in the non-LAST half-sweeps: A/B + tests
for V in 0 524288; do
  echo "255 n60 B16 v2off=$V: $(RBS_DISABLE_V2=$V timeout 600 python tools/prof_3d.py --m 255 --n 60 --random-basis --iters 3 2>/dev/null)"
done
timeout 1500 python -m pytest tests/test_gpu_zmarch.py tests/test_gpu_cases.py -x -q > gpurun_out/rc_tests.log 2>&1; tail -2 gpurun_out/rc_tests.log
timeout 1500 python -m pytest tests -m gpu -x -q -k "3 or three or c4 or edge or next3" > gpurun_out/rc_tests3d.log 2>&1; tail -2 gpurun_out/rc_tests3d.log
