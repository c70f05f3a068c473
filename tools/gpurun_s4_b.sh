# k_gsz<ZERO> (the symmetric preconditioner's pre-sweep from y = 0 without the fill and the y tiles):
# parity tests, A/B at 255^3 (RBS_DISABLE_V2 bit 20 keeps the k_fill_batch + half-sweep pair), c5 line
timeout 1500 python -m pytest tests/test_gpu_zmarch.py tests/test_gpu_next3.py tests/test_gpu_c5.py tests/test_gpu_parity.py::test_jacobi_smoother -q > gpurun_out/s4_zero_tests.log 2>&1; tail -2 gpurun_out/s4_zero_tests.log
for CFG in "--B 8 --n 40" "--B 16 --n 60"; do
  for V in 0 1048576; do
    echo "255 $CFG precond=sym v2off=$V: $(RBS_DISABLE_V2=$V timeout 600 python tools/prof_3d.py --m 255 $CFG --random-basis --iters 3 --precond 1 2>/dev/null)"
  done
done | tee gpurun_out/s4_zero_ab.txt
timeout 2400 python bench.py --config c5 --steps 1 --warmup 1 --precond sym > gpurun_out/s4_c5_sym.json 2> gpurun_out/s4_c5_sym.err
tail -1 gpurun_out/s4_c5_sym.json | cut -c1-300
