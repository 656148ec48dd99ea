# round 2, trip 7: F64S with spread-based plan reuse + K4 on the measured plan
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_softmin.py tests/test_gpu_solver.py tests/test_gpu_integration.py -q -m gpu -p no:cacheprovider -k "f64s or block_sparse or plan_reuse or integration or law" > gpurun_out/t10.log 2>&1; echo rc=$? >> gpurun_out/t10.log
timeout 1200 python tools/solve_bench.py c5 262144 2 > gpurun_out/c5_2step_f64s_b.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"softmin|f64s|plan_reduce" --csv --log-file gpurun_out/c5_launches_b.csv python tools/solve_bench.py c5 262144 1 > gpurun_out/ncu_c5b.log 2>&1
tail -n 3 gpurun_out/t10.log gpurun_out/c5_2step_f64s_b.log
