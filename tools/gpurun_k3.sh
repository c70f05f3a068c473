# K3 loads-first restructure: per-class times + graph iteration at c2, c2/c1 parity
python tools/prof_c2.py --build /tmp/c2basis.pt > /dev/null 2>&1
echo "c2: $(PROF_GRAPH=1 python tools/prof_c2.py --load /tmp/c2basis.pt --iters 20 | tr '\n' ' ')"
echo "c2 rbi: $(PROF_GRAPH=1 python tools/prof_c2.py --load /tmp/c2basis.pt --iters 20 --method rbi | tr '\n' ' ')"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -x -q > gpurun_out/k3_tests.log 2>&1; tail -1 gpurun_out/k3_tests.log
