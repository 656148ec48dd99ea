# session 3: experiment: 32-row groups for 16 <= kd < 64 with 64-column stages
timeout 900 python -m pytest tests/test_gpu_softmin.py tests/test_gpu_solver.py -q -m gpu -p no:cacheprovider -x -k "f64s or solver" > gpurun_out/s3_25_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s3_25_tests.log | cut -c1-300
timeout 600 python tools/solve_bench.py c5 262144 10 > gpurun_out/s3_25_c5.log 2>&1
python -c "
import json
for f in ('gpurun_out/s3_25_c5.log',):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(d['config'], d['seconds'], d['step_seconds'], d['objectives'][-1])"
