# z-march v2: parity (full GPU suite), A/B timings at 255^3, c2 bench line
timeout 600 python tools/prof_3d.py --m 255 --n 60 --random-basis --iters 3 > gpurun_out/z2_prof_255.json 2> gpurun_out/z2_prof.err
echo "m=255 new: $(cat gpurun_out/z2_prof_255.json)"
timeout 1500 python -m pytest tests/test_gpu_zmarch.py -x -q > gpurun_out/z2_tests.log 2>&1; tail -2 gpurun_out/z2_tests.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/z2_gpu_tests.log 2>&1; tail -2 gpurun_out/z2_gpu_tests.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/z2_bench.json 2> gpurun_out/z2_bench.err
tail -1 gpurun_out/z2_bench.json | cut -c1-300
