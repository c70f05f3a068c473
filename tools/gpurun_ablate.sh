# k_smooth3 ablations (RBS_DISABLE_V2 bits 12+: 1 no DMMA, 2 no sweeps, 4 no outputs)
python tools/prof_c2.py --build /tmp/c2basis.pt > /dev/null 2>&1
for d in 0 3 7 8 15 11; do
  echo "dbg=$d $(RBS_DISABLE_V2=$((d << 12)) python tools/prof_c2.py --load /tmp/c2basis.pt --iters 20 --method rbi)"
done
echo "v2 $(RBS_DISABLE_V2=2048 python tools/prof_c2.py --load /tmp/c2basis.pt --iters 20 --method rbi)"
