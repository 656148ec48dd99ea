# session 3: after the f64s_probe refactor: probe tests on both probes, f64s suite
timeout 900 python -m pytest tests/test_gpu_softmin.py tests/test_gpu_solver.py -q -m gpu -p no:cacheprovider -x -k "f64s or solver or c1" > gpurun_out/s3_39_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s3_39_tests.log | cut -c1-300
