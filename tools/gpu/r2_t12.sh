python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/t12.log 2>&1; echo rc=$? >> gpurun_out/t12.log
timeout 1500 python tools/solve_bench.py c5 262144 10 > gpurun_out/c5_full.log 2>&1
timeout 1500 python tools/solve_bench.py c4 1048576 10 > gpurun_out/c4_full.log 2>&1
tail -n 5 gpurun_out/t12.log; cat gpurun_out/c5_full.log gpurun_out/c4_full.log
