# guarded Jacobi copy-back (k_copy_unless_done): every Jacobi test + the smoother / edge / NEXT(3) files, then smoke
timeout 800 python -m pytest tests -m gpu -q -k "jacobi or smoother or edge or next3" > gpurun_out/s4e_tests.log 2>&1; tail -2 gpurun_out/s4e_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
