# ncu --set full of the half-sweeps of the symmetric preconditioner at 255^3 (B = 8, n = 40: c5's batch and width):
# k_gsz<8,0,0,1> (ZERO, from y = 0) next to k_gsz<8,0,0,0> / <8,1,0,0>
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "solve/" -k regex:'k_gsz|k_fill_batch' -c 20 \
    -o /tmp/z0 -f python tools/prof_3d.py --m 255 --B 8 --n 40 --random-basis --iters 2 --precond 1 --prof-only > gpurun_out/s4_z0_ncu.log 2>&1
python tools/ncu_brief.py /tmp/z0.ncu-rep > gpurun_out/s4_z0_brief.txt 2>&1; cat gpurun_out/s4_z0_brief.txt
