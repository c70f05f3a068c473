set -x
python tools/prof_c2.py --build /tmp/c2basis.pt > gpurun_out/r2_prof_build.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_smooth' -c 2 -o gpurun_out/r2_s3 python tools/prof_c2.py --load /tmp/c2basis.pt --iters 2 > gpurun_out/r2_ncu_s3.log 2>&1
RBS_DISABLE_V2=2048 ncu --set full --clock-control none --import-source on -k regex:'k_smooth' -c 2 -o gpurun_out/r2_s2 python tools/prof_c2.py --load /tmp/c2basis.pt --iters 2 > gpurun_out/r2_ncu_s2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_march3.py -x -q > gpurun_out/r2_m3_tests.log 2>&1
