# session 3: fp16-operand tcgen05 split: accuracy vs tf32/f64, tests on the tc path, timing sweep
timeout 300 python tools/tc_kind_check.py > gpurun_out/s3_tc_kind.log 2>&1; cat gpurun_out/s3_tc_kind.log | tail -12
timeout 900 python -m pytest tests/test_gpu_softmin.py tests/test_gpu_dist.py tests/test_gpu_sinkhorn.py -q -m gpu -p no:cacheprovider -x -k "low_rank or c2 or tc or partial or sinkhorn" > gpurun_out/s3_tc_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/s3_tc_tests.log
timeout 600 python tools/sweep_paths.py 1048576 5 "C2 K=16 prec=2" > gpurun_out/s3_sweep_kind.log 2>&1; cat gpurun_out/s3_sweep_kind.log
