# c5 N=1 reference solve on the z-plane marches: the paper's preconditioner and the symmetric one
timeout 2400 python bench.py --config c5 --steps 1 --warmup 0 --precond sym > gpurun_out/c5_sym.json 2> gpurun_out/c5_sym.err
tail -1 gpurun_out/c5_sym.json | cut -c1-300
