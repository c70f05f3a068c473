# c5 N=1 on the final build (symmetric preconditioner: z-march residual-projection)
mkdir -p gpurun_out
timeout 2400 python bench.py --config c5 --steps 2 --warmup 1 --precond sym > gpurun_out/h_c5_sym.json 2> gpurun_out/h_c5_sym.err
echo "c5 rc=$?"; tail -1 gpurun_out/h_c5_sym.json | cut -c1-300
