# round 2, trip 5: CNTGW_F64S measured-plan path
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_softmin.py -q -x -m gpu -p no:cacheprovider -k "f64s" > gpurun_out/t8.log 2>&1; echo rc=$? >> gpurun_out/t8.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_integration.py -q -s -m gpu -p no:cacheprovider -k "c5 or integration" > gpurun_out/t9.log 2>&1; echo rc=$? >> gpurun_out/t9.log
timeout 1200 python tools/solve_bench.py c5 262144 2 > gpurun_out/c5_2step_f64s.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"softmin|f64s|plan_reduce" --csv --log-file gpurun_out/c5_launches.csv python tools/solve_bench.py c5 262144 1 > gpurun_out/ncu_c5.log 2>&1
tail -n 3 gpurun_out/t8.log gpurun_out/t9.log gpurun_out/c5_2step_f64s.log
