# session 3: vanishing dot term (Gamma = 0) fast path in the F64S sweep: tests, solve times
timeout 900 python -m pytest tests/test_gpu_softmin.py tests/test_gpu_solver.py tests/test_gpu_fullsize.py -q -m gpu -p no:cacheprovider -x -k "f64s or solver or fullsize or full_size" > gpurun_out/s3_26_tests.log 2>&1; echo "tests rc=$?"; tail -12 gpurun_out/s3_26_tests.log | cut -c1-300
timeout 300 python tools/solve_bench.py c4 1048576 10 > gpurun_out/s3_26_c4.log 2>&1
timeout 200 python tools/solve_bench.py c5 262144 10 > gpurun_out/s3_26_c5.log 2>&1
python -c "
import json
for f in ('gpurun_out/s3_26_c4.log','gpurun_out/s3_26_c5.log'):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(d['config'], d['seconds'], d['step_seconds'], d['objectives'][-1])"
timeout 600 python tools/f64s_trace.py 1048576 0 14 c4 > gpurun_out/s3_26_trace_c4.log 2>&1; tail -5 gpurun_out/s3_26_trace_c4.log
