timeout 1500 python tools/solve_bench.py c4 1048576 10 > gpurun_out/c4_steps.log 2>&1
timeout 1500 python tools/solve_bench.py c5 262144 10 > gpurun_out/c5_steps.log 2>&1
python -c "
import json
for f in ('gpurun_out/c4_steps.log','gpurun_out/c5_steps.log'):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(d['config'], d['seconds'], d['step_seconds'])"
