# k_wtr v2 A/B at 255^3 n=60 and 511^3-like widths, 3D tests
timeout 600 python tools/prof_3d.py --m 255 --n 60 --random-basis --iters 3 > gpurun_out/w_prof_255.json 2> gpurun_out/w_prof.err
echo "m=255 n=60 B=16: $(cat gpurun_out/w_prof_255.json)"
timeout 600 python tools/prof_3d.py --m 255 --n 40 --B 8 --random-basis --iters 3 > gpurun_out/w_prof_255b8.json 2>> gpurun_out/w_prof.err
echo "m=255 n=40 B=8: $(cat gpurun_out/w_prof_255b8.json)"
timeout 1500 python -m pytest tests -m gpu -x -q -k "3 or three or c4 or slab or next3 or case or edge or zmarch" > gpurun_out/w_tests3d.log 2>&1; tail -2 gpurun_out/w_tests3d.log
