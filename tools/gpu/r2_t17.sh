python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench_r2.log 2>&1; echo rc=$? >> gpurun_out/bench_r2.log
tail -n 2 gpurun_out/bench_r2.log
