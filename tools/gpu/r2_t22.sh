python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_softmin.py tests/test_gpu_solver.py -q -m gpu -p no:cacheprovider -k "f64s or block_sparse" > gpurun_out/t22.log 2>&1; echo rc=$? >> gpurun_out/t22.log
timeout 1200 python tools/f64s_trace.py 1048576 2 20 c4 > gpurun_out/f64s_trace_c4d.log 2>&1
timeout 1500 python tools/solve_bench.py c4 1048576 10 > gpurun_out/c4_part.log 2>&1
timeout 1500 python tools/solve_bench.py c5 262144 10 > gpurun_out/c5_part.log 2>&1
tail -n 2 gpurun_out/t22.log; cat gpurun_out/f64s_trace_c4d.log gpurun_out/c4_part.log gpurun_out/c5_part.log
