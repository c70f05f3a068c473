# z-march v3: A/B timings at 255^3, then the new parity tests and the 3D GPU tests
timeout 600 python tools/prof_3d.py --m 255 --n 60 --random-basis --iters 3 > gpurun_out/z3_prof_255.json 2> gpurun_out/z3_prof.err
echo "m=255 new: $(cat gpurun_out/z3_prof_255.json)"; tail -3 gpurun_out/z3_prof.err
timeout 600 python tools/prof_3d.py --m 127 --n 20 --random-basis --iters 3 > gpurun_out/z3_prof_127.json 2>> gpurun_out/z3_prof.err
echo "m=127 new: $(cat gpurun_out/z3_prof_127.json)"
timeout 1500 python -m pytest tests/test_gpu_zmarch.py -x -q > gpurun_out/z3_tests.log 2>&1; tail -2 gpurun_out/z3_tests.log
timeout 1500 python -m pytest tests -m gpu -x -q -k "3 or three or c4 or slab or next3 or case or edge" > gpurun_out/z3_tests3d.log 2>&1; tail -2 gpurun_out/z3_tests3d.log
