# round 2: bench (both arms) + launch lists + ncu of the new kernels
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench_r2.log 2>&1; echo rc=$? >> gpurun_out/bench_r2.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r2.log 2>&1; echo rc=$? >> gpurun_out/bench_ref_r2.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-solve --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:softmin_f64s --launch-skip 24 --launch-count 1 -o gpurun_out/r2_ncu_f64s_c5_sparse python tools/f64s_trace.py 262144 0 14 c5 > gpurun_out/ncu_f64s.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:softmin_f64s --launch-skip 0 --launch-count 1 -o gpurun_out/r2_ncu_f64s_c5_measure python tools/f64s_trace.py 262144 0 2 c5 > gpurun_out/ncu_f64s_m.log 2>&1
tail -n 3 gpurun_out/bench_r2.log gpurun_out/bench_ref_r2.log gpurun_out/ncu_f64s.log
