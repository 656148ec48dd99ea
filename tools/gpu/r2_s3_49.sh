timeout 900 python -m pytest tests/test_gpu_native_solve.py -q -m gpu -p no:cacheprovider -x > gpurun_out/s3_49_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s3_49_tests.log | cut -c1-300
