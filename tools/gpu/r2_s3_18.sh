# session 3: F64S sweeps without L2 column chunks: f64s tests, step times
timeout 900 python -m pytest tests/test_gpu_softmin.py tests/test_gpu_solver.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -q -m gpu -p no:cacheprovider -x -k "f64s or solver or fullsize or full_size or partial" > gpurun_out/s3_18_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s3_18_tests.log | cut -c1-300
timeout 900 python tools/solve_bench.py c4 1048576 10 > gpurun_out/s3_18_c4.log 2>&1
timeout 600 python tools/solve_bench.py c5 262144 10 > gpurun_out/s3_18_c5.log 2>&1
python -c "
import json
for f in ('gpurun_out/s3_18_c4.log','gpurun_out/s3_18_c5.log'):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(d['config'], d['seconds'], d['step_seconds'], d['objectives'][-1])"
timeout 600 python tools/f64s_trace.py 1048576 3 12 c4 > gpurun_out/s3_18_trace_c4.log 2>&1; head -12 gpurun_out/s3_18_trace_c4.log
