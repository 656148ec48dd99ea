# session 3: bias-only column update within a loop (cntgw_update_cols_f64s): full GPU suite, solve times
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/s3_35_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s3_35_tests.log | cut -c1-300
timeout 300 python tools/solve_bench.py c4 1048576 10 > gpurun_out/s3_35_c4.log 2>&1
timeout 200 python tools/solve_bench.py c5 262144 10 > gpurun_out/s3_35_c5.log 2>&1
python -c "
import json
for f in ('gpurun_out/s3_35_c4.log','gpurun_out/s3_35_c5.log'):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(d['config'], d['seconds'], d['step_seconds'], d['objectives'][-1])"
