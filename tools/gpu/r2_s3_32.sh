# session 3: per-warp stage skipping in the sparse K4 (plan_reduce on the F64S plan): K4 / solver / api / fullsize tests, C4 and C5 solve times
timeout 1500 python -m pytest tests/test_gpu_solver.py tests/test_gpu_api.py tests/test_gpu_fullsize.py tests/test_gpu_native_solve.py tests/test_gpu_divergence.py tests/test_gpu_dist.py -q -m gpu -p no:cacheprovider -x > gpurun_out/s3_32_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s3_32_tests.log | cut -c1-300
timeout 300 python tools/solve_bench.py c4 1048576 10 > gpurun_out/s3_32_c4.log 2>&1
timeout 200 python tools/solve_bench.py c5 262144 10 > gpurun_out/s3_32_c5.log 2>&1
python -c "
import json
for f in ('gpurun_out/s3_32_c4.log','gpurun_out/s3_32_c5.log'):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(d['config'], d['seconds'], d['step_seconds'], d['objectives'])"
