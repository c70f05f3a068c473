# final round-2 measurements, part A: c2 bench line (driver-equivalent), reference arm, c1, RBI,
# Case 1/2, launch list and the ncu --set full capture of the c2 kernels (traffic JSON)
python bench.py --steps 20 --warmup 5 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
tail -1 gpurun_out/final_bench.json | cut -c1-300
python bench.py --config c1 --steps 20 --warmup 5 > gpurun_out/final_c1.json 2> gpurun_out/final_c1.err
python bench.py --method rbi --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/final_rbi.json 2> gpurun_out/final_rbi.err
python bench.py --config case1 --steps 6 --warmup 3 > gpurun_out/final_case1.json 2> gpurun_out/final_case1.err
python bench.py --config case2 --steps 6 --warmup 3 > gpurun_out/final_case2.json 2> gpurun_out/final_case2.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
tail -1 gpurun_out/final_ref.json | cut -c1-200
# launch list of the timed region (one batch stream: ncu serialises kernels anyway)
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --streams 1 \
    > gpurun_out/final_launches.log 2>&1
# ncu --set full of the four c2 kernels, exactly as bench.py launches them (tools/prof_c2.py: same
# kernels and launch configuration, eager), summarised on the box
python tools/prof_c2.py --build /tmp/c2basis.pt > /dev/null 2>&1
ncu --set full --clock-control none -k regex:'k_smooth2|k_cgp2|k_resid2|k_reduce_solve' -c 8 -o /tmp/final_c2 -f \
    python tools/prof_c2.py --load /tmp/c2basis.pt --iters 2 > gpurun_out/final_ncu.log 2>&1
python tools/ncu_brief.py /tmp/final_c2.ncu-rep > gpurun_out/final_ncu_brief.txt 2>&1
python tools/ncu_summary.py /tmp/final_c2.ncu-rep > gpurun_out/final_ncu_summary.md 2>&1
python tools/ncu_traffic.py /tmp/final_c2.ncu-rep gpurun_out/final_traffic.json \
    "-k regex:'k_smooth2|k_cgp2|k_resid2|k_reduce_solve' -c 8, python tools/prof_c2.py --load basis --iters 2 (c2, B=32, n=40)" > /dev/null 2>&1
cat gpurun_out/final_ncu_brief.txt
