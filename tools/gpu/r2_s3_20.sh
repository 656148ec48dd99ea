# session 3: probe bound test; C5 with 64-row groups (CNTGW_F64S_RG=2) against the default 128
timeout 600 python -m pytest tests/test_gpu_softmin.py -q -m gpu -p no:cacheprovider -x -k "probe_bounds" > gpurun_out/s3_20_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/s3_20_tests.log | cut -c1-400
CNTGW_F64S_RG=2 timeout 600 python tools/solve_bench.py c5 262144 10 > gpurun_out/s3_20_c5_rg2.log 2>&1
timeout 600 python tools/solve_bench.py c5 262144 10 > gpurun_out/s3_20_c5.log 2>&1
python -c "
import json
for f in ('gpurun_out/s3_20_c5_rg2.log','gpurun_out/s3_20_c5.log'):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d['config'], d['seconds'], d['step_seconds'], d['objectives'][-1])"
CNTGW_F64S_RG=2 timeout 600 python tools/f64s_trace.py 262144 3 12 c5 > gpurun_out/s3_20_trace_c5_rg2.log 2>&1; tail -4 gpurun_out/s3_20_trace_c5_rg2.log
