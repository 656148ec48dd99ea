python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/t24.log 2>&1; echo rc=$? >> gpurun_out/t24.log
timeout 1200 python bench.py > gpurun_out/bench_r2b.log 2>&1; echo rc=$? >> gpurun_out/bench_r2b.log
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"plan_reduce|f64s|softmin|select" --csv --log-file gpurun_out/r2_c4_step_launches.csv python tools/solve_bench.py c4 1048576 2 > gpurun_out/ncu_c4step2.log 2>&1
grep -E "passed|failed" gpurun_out/t24.log | tail -2; tail -n 2 gpurun_out/smoke.log; tail -n 2 gpurun_out/bench_r2b.log | cut -c1-400
