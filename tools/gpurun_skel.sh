python tools/prof_c2.py --build /tmp/c2basis.pt > /dev/null 2>&1
RBS_DISABLE_V2=$((15 << 12)) ncu --set full --clock-control none -k regex:k_smooth3 -c 1 -o /tmp/sk -f python tools/prof_c2.py --load /tmp/c2basis.pt --iters 2 --method rbi > gpurun_out/sk_ncu.log 2>&1
python tools/ncu_brief.py /tmp/sk.ncu-rep
ncu -i /tmp/sk.ncu-rep --page details --csv 2>/dev/null | grep -E "Elapsed Cycles|SM Active Cycles|Duration|Executed Ipc|Issue Slots Busy|Registers Per|Achieved Occupancy|Waves Per SM|Grid Size|Block Size|Dynamic Shared|No Eligible|Active Warps Per" | cut -c1-200
python tools/ncu_lines.py /tmp/sk.ncu-rep k_smooth3 25
