# session 3: 64-column stages probed two per 128-column MMA tile; hoisting equivalence test: f64s tests, C5/C4 traces and solve times
timeout 900 python -m pytest tests/test_gpu_softmin.py tests/test_gpu_solver.py tests/test_gpu_fullsize.py -q -m gpu -p no:cacheprovider -x -k "f64s or solver or fullsize or full_size" > gpurun_out/s3_36_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s3_36_tests.log | cut -c1-300
timeout 300 python tools/f64s_trace.py 262144 3 3 c5 > gpurun_out/s3_36_trace_c5.log 2>&1; head -3 gpurun_out/s3_36_trace_c5.log
timeout 200 python tools/solve_bench.py c5 262144 10 > gpurun_out/s3_36_c5.log 2>&1
timeout 300 python tools/solve_bench.py c4 1048576 10 > gpurun_out/s3_36_c4.log 2>&1
python -c "
import json
for f in ('gpurun_out/s3_36_c4.log','gpurun_out/s3_36_c5.log'):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(d['config'], d['seconds'], d['step_seconds'], d['objectives'][-1])"
