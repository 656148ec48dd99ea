# session 3: column-split probe epilogue (16 warps) at 256-column stages: probe tests, traces, C4/C5 step times
timeout 600 python -m pytest tests/test_gpu_softmin.py tests/test_gpu_solver.py -q -m gpu -p no:cacheprovider -x -k "f64s or solver" > gpurun_out/s3_16_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s3_16_tests.log | cut -c1-300
timeout 600 python tools/f64s_trace.py 1048576 0 12 c4 > gpurun_out/s3_16_trace_c4.log 2>&1; head -12 gpurun_out/s3_16_trace_c4.log
timeout 600 python tools/f64s_trace.py 262144 1 8 c5 > gpurun_out/s3_16_trace_c5.log 2>&1; head -8 gpurun_out/s3_16_trace_c5.log
timeout 900 python tools/solve_bench.py c4 1048576 10 > gpurun_out/s3_16_c4.log 2>&1
timeout 600 python tools/solve_bench.py c5 262144 10 > gpurun_out/s3_16_c5.log 2>&1
python -c "
import json
for f in ('gpurun_out/s3_16_c4.log','gpurun_out/s3_16_c5.log'):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(d['config'], d['seconds'], d['step_seconds'], d['objectives'][-1])"
