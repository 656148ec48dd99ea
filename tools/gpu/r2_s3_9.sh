# session 3: sweep threshold 2^-48 + halving/doubling re-measurement interval: f64s tests, C4/C5 step times, per-sweep trace
timeout 900 python -m pytest tests/test_gpu_softmin.py tests/test_gpu_fullsize.py -q -m gpu -p no:cacheprovider -x -k "f64s or fullsize or full_size" > gpurun_out/s3_9_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s3_9_tests.log
timeout 900 python tools/solve_bench.py c4 1048576 10 > gpurun_out/s3_9_c4.log 2>&1
timeout 600 python tools/solve_bench.py c5 262144 10 > gpurun_out/s3_9_c5.log 2>&1
python -c "
import json
for f in ('gpurun_out/s3_9_c4.log','gpurun_out/s3_9_c5.log'):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(d['config'], d['seconds'], d['step_seconds'], d['objectives'][-1])"
timeout 600 python tools/f64s_trace.py 1048576 3 40 c4 > gpurun_out/s3_9_trace_c4.log 2>&1; head -24 gpurun_out/s3_9_trace_c4.log
timeout 600 python tools/f64s_trace.py 262144 3 40 c5 > gpurun_out/s3_9_trace_c5.log 2>&1; head -24 gpurun_out/s3_9_trace_c5.log
