# quick K3 A/B on the GPU: GPU tests (TESTK: -k filter), then per-class times of one c2 batch (eager
# profile mode); NCU=1: one ncu --set full capture of k_smooth2, summarised on the box
# (the raw report of the full module is > 64 MiB, it is not copied back)
timeout 900 python -m pytest tests -m gpu -x -q ${TESTK:+-k "$TESTK"} > gpurun_out/q_tests.log 2>&1
tail -1 gpurun_out/q_tests.log
python tools/prof_c2.py --build /tmp/c2basis.pt > gpurun_out/q_build.log 2>&1
python tools/prof_c2.py --load /tmp/c2basis.pt --iters 30 | tee gpurun_out/q_v3.log
RBS_DISABLE_V2=${AB:-4096} python tools/prof_c2.py --load /tmp/c2basis.pt --iters 30 | tee gpurun_out/q_v2.log
if [ -n "$NCU" ]; then
  ncu --set full --clock-control none --import-source on -k regex:${NCUK:-k_smooth2} -c 1 -o /tmp/q_s3 -f python tools/prof_c2.py --load /tmp/c2basis.pt --iters 2 > gpurun_out/q_ncu.log 2>&1
  python tools/ncu_brief.py /tmp/q_s3.ncu-rep > gpurun_out/q_ncu_brief.txt 2>&1
  python tools/ncu_lines.py /tmp/q_s3.ncu-rep ${NCUK:-k_smooth2} 45 > gpurun_out/q_ncu_lines.txt 2>&1
  cat gpurun_out/q_ncu_brief.txt
fi
