# z-march check: new parity tests, the 3D GPU tests, A/B timings at 127^3 and 255^3
timeout 1200 python -m pytest tests/test_gpu_zmarch.py -x -q > gpurun_out/z_tests.log 2>&1; tail -3 gpurun_out/z_tests.log
timeout 1500 python -m pytest tests -m gpu -x -q -k "3 or three or c4 or slab or next3 or case or edge" > gpurun_out/z_tests3d.log 2>&1; tail -2 gpurun_out/z_tests3d.log
for M in 127 255; do
  N=20; [ $M = 255 ] && N=60
  timeout 600 python tools/prof_3d.py --m $M --n $N --random-basis --iters 3 > gpurun_out/z_prof_$M.json 2> gpurun_out/z_prof_$M.err
  RBS_DISABLE_V2=65536 timeout 600 python tools/prof_3d.py --m $M --n $N --random-basis --iters 3 > gpurun_out/z_prof_${M}_old.json 2>> gpurun_out/z_prof_$M.err
  echo "m=$M new: $(cat gpurun_out/z_prof_$M.json)"; echo "m=$M old: $(cat gpurun_out/z_prof_${M}_old.json)"
done
