# session-4 final: smoke + the full GPU suite on the final build (Jacobi fix, k_gsz<ZERO>)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s4f_smoke.log 2>&1; tail -1 gpurun_out/s4f_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s4f_gpu_tests.log 2>&1; tail -2 gpurun_out/s4f_gpu_tests.log
