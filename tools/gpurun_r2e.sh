# round-2 end (session 3): GPU suite on the restored build, c4 line with k_prolz, c5 N=1 on the z-plane marches
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/e_gpu_tests.log 2>&1; tail -2 gpurun_out/e_gpu_tests.log
timeout 1200 python bench.py --config c4 --queries 64 --steps 1 --warmup 1 > gpurun_out/e_c4.json 2> gpurun_out/e_c4.err
tail -1 gpurun_out/e_c4.json | cut -c1-300
timeout 2400 python bench.py --config c5 --steps 2 --warmup 1 --precond sym > gpurun_out/e_c5_sym.json 2> gpurun_out/e_c5_sym.err
tail -1 gpurun_out/e_c5_sym.json | cut -c1-300
