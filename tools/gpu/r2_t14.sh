python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_softmin.py tests/test_gpu_solver.py tests/test_gpu_fullsize.py -q -m gpu -p no:cacheprovider -k "f64s or block_sparse or c5" > gpurun_out/t14.log 2>&1; echo rc=$? >> gpurun_out/t14.log
timeout 1200 python tools/f64s_trace.py 1048576 2 40 c4 > gpurun_out/f64s_trace_c4b.log 2>&1
timeout 1200 python tools/f64s_trace.py 262144 1 40 c5 > gpurun_out/f64s_trace_c5b.log 2>&1
timeout 1500 python tools/solve_bench.py c5 262144 10 > gpurun_out/c5_full_b.log 2>&1
CNTGW_PRECISION=f64s timeout 1500 python tools/solve_bench.py c4 1048576 10 > gpurun_out/c4_full_f64s.log 2>&1
tail -n 2 gpurun_out/t14.log; grep -E "sweep (1|2|8|9|20|40):" gpurun_out/f64s_trace_c4b.log gpurun_out/f64s_trace_c5b.log; cat gpurun_out/c5_full_b.log gpurun_out/c4_full_f64s.log
