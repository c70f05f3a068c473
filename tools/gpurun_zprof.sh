# ncu of the 3D passes at 255^3 (n = 60, B = 16, random orthonormal basis), one RBCG iteration
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "solve/" -k regex:'k_gsz|k_cgz|k_xrz|k_wtr|k_proj|k_prolong|k_reduce' -c 8 \
    -o /tmp/z255 -f python tools/prof_3d.py --m 255 --n 60 --random-basis --iters 1 --prof-only > gpurun_out/zp_ncu.log 2>&1
python tools/ncu_brief.py /tmp/z255.ncu-rep > gpurun_out/zp_brief.txt 2>&1; cat gpurun_out/zp_brief.txt
for K in k_gsz k_cgz k_xrz; do python tools/ncu_lines.py /tmp/z255.ncu-rep $K 40 > gpurun_out/zp_lines_$K.txt 2>&1; done
ncu -i /tmp/z255.ncu-rep --page details --csv > gpurun_out/zp_details.csv 2>&1
