# session-3 diagnostics: per-step solve times, kernel shares of 3 outer steps at C4/C5, pipe peaks, tc variants
timeout 900 python tools/solve_bench.py c4 1048576 10 > gpurun_out/s3_c4_steps.log 2>&1
timeout 600 python tools/solve_bench.py c5 262144 10 > gpurun_out/s3_c5_steps.log 2>&1
python -c "
import json
for f in ('gpurun_out/s3_c4_steps.log','gpurun_out/s3_c5_steps.log'):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(d['config'], d['seconds'], d['step_seconds'], d['objectives'][-1])"
./tools/ubench_pipes > gpurun_out/s3_pipes.log 2>&1; cat gpurun_out/s3_pipes.log
timeout 600 python tools/sweep_paths.py 1048576 5 > gpurun_out/s3_sweep_paths.log 2>&1; tail -20 gpurun_out/s3_sweep_paths.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/s3_c4_launches.csv python tools/solve_bench.py c4 1048576 3 > gpurun_out/s3_c4_ncu.log 2>&1; echo "ncu c4 rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/s3_c5_launches.csv python tools/solve_bench.py c5 262144 3 > gpurun_out/s3_c5_ncu.log 2>&1; echo "ncu c5 rc=$?"
