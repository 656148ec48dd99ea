# session 3: re-probe when the re-vote keeps > 25%: f64s tests, C4 step times, Gamma = 0 trace
timeout 900 python -m pytest tests/test_gpu_softmin.py tests/test_gpu_fullsize.py tests/test_gpu_solver.py -q -m gpu -p no:cacheprovider -x -k "f64s or fullsize or full_size or solver" > gpurun_out/s3_11_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s3_11_tests.log
timeout 900 python tools/solve_bench.py c4 1048576 10 > gpurun_out/s3_11_c4.log 2>&1
python -c "
import json
for f in ('gpurun_out/s3_11_c4.log',):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(d['config'], d['seconds'], d['step_seconds'], d['objectives'][-1])"
timeout 600 python tools/f64s_trace.py 1048576 0 16 c4 > gpurun_out/s3_11_trace_c4.log 2>&1; head -16 gpurun_out/s3_11_trace_c4.log
timeout 600 python tools/f64s_trace.py 1048576 1 16 c4 > gpurun_out/s3_11_trace_c4_1.log 2>&1; head -16 gpurun_out/s3_11_trace_c4_1.log
