# round 2, trip 2: block-sparse K4, fixed tests, C4 step timing
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_fullsize.py -q -s -m gpu -p no:cacheprovider > gpurun_out/t3.log 2>&1; echo rc=$? >> gpurun_out/t3.log
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_softmin.py -q -s -m gpu -p no:cacheprovider -k "sparse or law or c3 or plan_reuse or block_sparse" > gpurun_out/t4.log 2>&1; echo rc=$? >> gpurun_out/t4.log
for S in 1 0; do CNTGW_K4_SPARSE=$S timeout 600 python tools/solve_bench.py c4 1048576 2 > gpurun_out/c4_2step_k4s$S.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"plan_reduce|ctr_plan" --csv --log-file gpurun_out/k4_launches.csv python tools/solve_bench.py c4 1048576 1 > gpurun_out/ncu_k4.log 2>&1
tail -n 3 gpurun_out/t3.log gpurun_out/t4.log gpurun_out/c4_2step_k4s*.log
