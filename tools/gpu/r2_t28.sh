timeout 900 python -m pytest tests/test_gpu_softmin.py -q -m gpu -p no:cacheprovider -x -k "f64s" > gpurun_out/t28_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t28_tests.log
timeout 600 python tools/f64s_trace.py 1048576 3 30 c4 > gpurun_out/f64s_trace_c4_probe.log 2>&1; head -12 gpurun_out/f64s_trace_c4_probe.log; tail -2 gpurun_out/f64s_trace_c4_probe.log
CNTGW_F64S_PROBE=0 timeout 600 python tools/f64s_trace.py 1048576 3 12 c4 > gpurun_out/f64s_trace_c4_noprobe.log 2>&1; head -12 gpurun_out/f64s_trace_c4_noprobe.log
timeout 900 python tools/solve_bench.py c4 1048576 10 > gpurun_out/c4_steps.log 2>&1
timeout 600 python tools/solve_bench.py c5 262144 10 > gpurun_out/c5_steps.log 2>&1
python -c "
import json
for f in ('gpurun_out/c4_steps.log','gpurun_out/c5_steps.log'):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(d['config'], d['seconds'], d['step_seconds'], d['objectives'][-1])"
