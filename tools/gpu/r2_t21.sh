python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python tools/solve_bench.py c4 1048576 10 > gpurun_out/c4_sel.log 2>&1
timeout 1500 python tools/solve_bench.py c5 262144 10 > gpurun_out/c5_sel.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_solver.py tests/test_gpu_dist.py tests/test_gpu_native_solve.py -q -m gpu -p no:cacheprovider > gpurun_out/t21.log 2>&1; echo rc=$? >> gpurun_out/t21.log
cat gpurun_out/c4_sel.log gpurun_out/c5_sel.log; tail -n 3 gpurun_out/t21.log
