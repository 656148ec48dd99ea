# session 3: experiment: 128-column stages for kd < 16 (C4), 8192-stage lists
timeout 900 python -m pytest tests/test_gpu_softmin.py tests/test_gpu_solver.py -q -m gpu -p no:cacheprovider -x -k "f64s or solver" > gpurun_out/s3_24_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s3_24_tests.log | cut -c1-300
timeout 900 python tools/solve_bench.py c4 1048576 10 > gpurun_out/s3_24_c4.log 2>&1
python -c "
import json
for f in ('gpurun_out/s3_24_c4.log',):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(d['config'], d['seconds'], d['step_seconds'], d['objectives'])"
timeout 600 python tools/f64s_trace.py 1048576 3 12 c4 > gpurun_out/s3_24_trace_c4.log 2>&1; cat gpurun_out/s3_24_trace_c4.log
