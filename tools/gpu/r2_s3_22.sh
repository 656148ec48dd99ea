# session 3: new F64S row-group defaults (32 rows for kd < 16, 64 rows for 16 <= kd < 64): full GPU suite, solve times
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/s3_22_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s3_22_tests.log | cut -c1-300
timeout 900 python tools/solve_bench.py c4 1048576 10 > gpurun_out/s3_22_c4.log 2>&1
timeout 600 python tools/solve_bench.py c5 262144 10 > gpurun_out/s3_22_c5.log 2>&1
python -c "
import json
for f in ('gpurun_out/s3_22_c4.log','gpurun_out/s3_22_c5.log'):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(d['config'], d['seconds'], d['step_seconds'], d['objectives'][-1])"
