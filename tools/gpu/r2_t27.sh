timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/t27_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/t27_tests.log
timeout 900 python tools/solve_bench.py c4 1048576 10 > gpurun_out/c4_steps.log 2>&1
timeout 600 python tools/solve_bench.py c5 262144 10 > gpurun_out/c5_steps.log 2>&1
python -c "
import json
for f in ('gpurun_out/c4_steps.log','gpurun_out/c5_steps.log'):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(d['config'], d['seconds'], d['step_seconds'], d['objectives'][-1])"
timeout 900 python bench.py > gpurun_out/t27_bench.log 2>&1; echo "bench rc=$?"; tail -c 3000 gpurun_out/t27_bench.log
