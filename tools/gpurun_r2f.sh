# N = 2 query-shard bench code path on a one-GPU box (gloo plumbing, both ranks on cuda:0:
# a smoke of the torchrun path, not a scaling number), then the driver-equivalent c2 line
mkdir -p gpurun_out
RBS_BENCH_SMOKE_1GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 2 --warmup 3 \
    > gpurun_out/f_n2_smoke.json 2> gpurun_out/f_n2_smoke.err
echo "n2 smoke rc=$?"; tail -1 gpurun_out/f_n2_smoke.json | cut -c1-400
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/f_c2.json 2> gpurun_out/f_c2.err
echo "c2 rc=$?"; tail -1 gpurun_out/f_c2.json | cut -c1-600
