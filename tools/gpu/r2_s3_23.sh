# session 3: 64-column stages for 16 <= kd < 64 (shared f64s_stage_cols): f64s / solver / fullsize tests, C5 solve
timeout 1200 python -m pytest tests/test_gpu_softmin.py tests/test_gpu_solver.py tests/test_gpu_fullsize.py tests/test_gpu_native_solve.py tests/test_gpu_dist.py -q -m gpu -p no:cacheprovider -x > gpurun_out/s3_23_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s3_23_tests.log | cut -c1-300
timeout 600 python tools/solve_bench.py c5 262144 10 > gpurun_out/s3_23_c5.log 2>&1
python -c "
import json
for f in ('gpurun_out/s3_23_c5.log',):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(d['config'], d['seconds'], d['step_seconds'], d['objectives'])"
timeout 600 python tools/f64s_trace.py 262144 3 12 c5 > gpurun_out/s3_23_trace_c5.log 2>&1; cat gpurun_out/s3_23_trace_c5.log
