# session 3: F64S rows gather hoisted out of the sweep loop: full GPU suite, solve times, traces still valid
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/s3_27_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s3_27_tests.log | cut -c1-300
timeout 300 python tools/solve_bench.py c4 1048576 10 > gpurun_out/s3_27_c4.log 2>&1
timeout 200 python tools/solve_bench.py c5 262144 10 > gpurun_out/s3_27_c5.log 2>&1
python -c "
import json
for f in ('gpurun_out/s3_27_c4.log','gpurun_out/s3_27_c5.log'):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(d['config'], d['seconds'], d['step_seconds'], d['objectives'][-1])"
timeout 300 python tools/f64s_trace.py 262144 3 6 c5 > gpurun_out/s3_27_trace_c5.log 2>&1; tail -3 gpurun_out/s3_27_trace_c5.log
