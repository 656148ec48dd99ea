python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_native_solve.py -q -m gpu -p no:cacheprovider > gpurun_out/t19.log 2>&1; echo rc=$? >> gpurun_out/t19.log
timeout 1200 python tools/f64s_trace.py 1048576 2 12 c4 > gpurun_out/f64s_trace_c4c.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"plan_reduce|f64s|softmin" --csv --log-file gpurun_out/c4_step_launches.csv python tools/solve_bench.py c4 1048576 1 > gpurun_out/ncu_c4step.log 2>&1
tail -n 2 gpurun_out/t19.log; cat gpurun_out/f64s_trace_c4c.log
