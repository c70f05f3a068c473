# round-2 end measurements (z-march build), part A: smoke, full GPU suite, c2 line, c2 launch list,
# ncu --set full of the c2 kernels (traffic JSON keyed on the instantiations), ncu of the 3D passes
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2z_smoke.log 2>&1; tail -1 gpurun_out/r2z_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2z_gpu_tests.log 2>&1; tail -2 gpurun_out/r2z_gpu_tests.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2z_bench.json 2> gpurun_out/r2z_bench.err
tail -1 gpurun_out/r2z_bench.json | cut -c1-300
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2z_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --streams 1 \
    > gpurun_out/r2z_launches.log 2>&1
python tools/launch_summary.py gpurun_out/r2z_launches.csv > gpurun_out/r2z_launches.md 2>&1; head -12 gpurun_out/r2z_launches.md
python tools/prof_c2.py --build /tmp/c2basis.pt > /dev/null 2>&1
ncu --set full --clock-control none -k regex:'k_smooth2|k_cgp2|k_resid2|k_reduce_solve' -c 8 -o /tmp/r2z_c2 -f \
    python tools/prof_c2.py --load /tmp/c2basis.pt --iters 2 > gpurun_out/r2z_ncu.log 2>&1
python tools/ncu_summary.py /tmp/r2z_c2.ncu-rep > gpurun_out/r2z_ncu_c2.md 2>&1
python tools/ncu_traffic.py /tmp/r2z_c2.ncu-rep gpurun_out/r2z_traffic.json \
    "-k regex:'k_smooth2|k_cgp2|k_resid2|k_reduce_solve' -c 8, python tools/prof_c2.py --load basis --iters 2 (c2, B=32, n=40)" > /dev/null 2>&1
ncu --set full --clock-control none --nvtx --nvtx-include "solve/" -k regex:'k_gsz|k_cgz|k_xrz|k_wtr|k_prolz|k_reduce' -c 8 \
    -o /tmp/r2z_3d -f python tools/prof_3d.py --m 255 --n 60 --random-basis --iters 1 --prof-only > gpurun_out/r2z_ncu3d.log 2>&1
python tools/ncu_summary.py /tmp/r2z_3d.ncu-rep > gpurun_out/r2z_ncu_3d.md 2>&1; head -20 gpurun_out/r2z_ncu_3d.md
