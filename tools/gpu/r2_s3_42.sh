# session 3: exact-scale guards (tc kernel NaN on impossible scales, probe stands down): tc + f64s tests
timeout 900 python -m pytest tests/test_gpu_softmin.py tests/test_gpu_sinkhorn.py tests/test_gpu_dist.py -q -m gpu -p no:cacheprovider -x > gpurun_out/s3_42_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s3_42_tests.log | cut -c1-300
