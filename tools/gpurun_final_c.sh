# final round-2 measurements, part C: c3 / c4 strong-scaling shards at N = 1 (fixed query sets)
timeout 1500 python bench.py --config c3 --queries 128 --steps 1 --warmup 1 > gpurun_out/final_c3.json 2> gpurun_out/final_c3.err
tail -1 gpurun_out/final_c3.json | cut -c1-200
timeout 1500 python bench.py --config c4 --queries 64 --steps 1 --warmup 1 > gpurun_out/final_c4.json 2> gpurun_out/final_c4.err
tail -1 gpurun_out/final_c4.json | cut -c1-200
