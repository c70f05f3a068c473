# TMA prolongation (k_prolz) A/B at 255^3 and 127^3, 3D tests
for V in 0 262144; do
  echo "255 n60 B16 v2off=$V: $(RBS_DISABLE_V2=$V timeout 600 python tools/prof_3d.py --m 255 --n 60 --random-basis --iters 3 2>/dev/null)"
done
echo "255 n40 B8: $(timeout 600 python tools/prof_3d.py --m 255 --n 40 --B 8 --random-basis --iters 3 2>/dev/null)"
timeout 1800 python -m pytest tests -m gpu -x -q -k "3 or three or c4 or slab or next3 or case or edge or zmarch" > gpurun_out/pz_tests3d.log 2>&1; tail -2 gpurun_out/pz_tests3d.log
