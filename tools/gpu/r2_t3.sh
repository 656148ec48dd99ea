# round 2, trip 3: fp64 K4 exponentials, native NCCL comm, partial-LSE tests
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_dist.py -q -s -m gpu -p no:cacheprovider > gpurun_out/t5.log 2>&1; echo rc=$? >> gpurun_out/t5.log
timeout 900 python -m pytest tests/test_gpu_solver.py -q -s -m gpu -p no:cacheprovider > gpurun_out/t6.log 2>&1; echo rc=$? >> gpurun_out/t6.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"plan_reduce" --csv --log-file gpurun_out/k4_launches2.csv python tools/solve_bench.py c4 1048576 2 > gpurun_out/ncu_k4b.log 2>&1
CNTGW_K4_SPARSE=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"plan_reduce" --csv --log-file gpurun_out/k4_launches2_dense.csv python tools/solve_bench.py c4 1048576 2 > gpurun_out/ncu_k4c.log 2>&1
tail -n 3 gpurun_out/t5.log gpurun_out/t6.log
