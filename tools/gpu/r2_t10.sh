python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python tools/f64s_trace.py 262144 1 140 > gpurun_out/f64s_trace2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_softmin.py tests/test_gpu_solver.py tests/test_gpu_integration.py tests/test_gpu_fullsize.py -q -m gpu -p no:cacheprovider -k "f64s or block_sparse or plan_reuse or integration or law or c5" > gpurun_out/t11.log 2>&1; echo rc=$? >> gpurun_out/t11.log
timeout 1500 python tools/solve_bench.py c5 262144 2 > gpurun_out/c5_2step_c.log 2>&1
grep -E "sweep (1|2|3|4|7|8|9|15|16|17|31|32|33|63|64|65|100|127|128|129|140):" gpurun_out/f64s_trace2.log; tail -n 3 gpurun_out/t11.log gpurun_out/c5_2step_c.log
