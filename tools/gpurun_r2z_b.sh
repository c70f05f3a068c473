# round-2 end measurements (z-march build), part B: the other configs and the reference arm,
# and one compute-sanitizer attempt on tiny solves
for T in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize_small.py > gpurun_out/r2z_sanitize_$T.log 2>&1
  echo "$T rc=$? $(tail -2 gpurun_out/r2z_sanitize_$T.log | tr '\n' ' ')"
done
python bench.py --config c1 --steps 20 --warmup 5 > gpurun_out/r2z_c1.json 2> gpurun_out/r2z_c1.err
python bench.py --method rbi --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/r2z_rbi.json 2> gpurun_out/r2z_rbi.err
python bench.py --config case1 --steps 6 --warmup 3 > gpurun_out/r2z_case1.json 2> gpurun_out/r2z_case1.err
python bench.py --config case2 --steps 6 --warmup 3 > gpurun_out/r2z_case2.json 2> gpurun_out/r2z_case2.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2z_ref.json 2> gpurun_out/r2z_ref.err
timeout 1500 python bench.py --config c4 --queries 64 --steps 1 --warmup 1 > gpurun_out/r2z_c4.json 2> gpurun_out/r2z_c4.err
timeout 1500 python bench.py --config c3 --queries 128 --steps 1 --warmup 1 > gpurun_out/r2z_c3.json 2> gpurun_out/r2z_c3.err
for f in c1 rbi case1 case2 ref c4 c3; do echo "$f: $(tail -1 gpurun_out/r2z_$f.json | cut -c1-160)"; done
timeout 2400 python bench.py --config c5 --steps 1 --warmup 0 --precond sym > gpurun_out/r2z_c5_sym.json 2> gpurun_out/r2z_c5_sym.err
echo "c5: $(tail -1 gpurun_out/r2z_c5_sym.json | cut -c1-160)"
