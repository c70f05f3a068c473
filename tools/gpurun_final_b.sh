# final round-2 measurements, part B: the GPU test suite and smoke (compute-sanitizer is closed on this pool)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/final_gpu_tests.log 2>&1; tail -2 gpurun_out/final_gpu_tests.log
