python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/t15.log 2>&1; echo rc=$? >> gpurun_out/t15.log
timeout 1500 python tools/solve_bench.py c5 262144 10 > gpurun_out/c5_full_c.log 2>&1
timeout 1500 python tools/solve_bench.py c4 1048576 10 > gpurun_out/c4_full_c.log 2>&1
timeout 600 python tools/solve_bench.py c3 > gpurun_out/c3_full_c.log 2>&1
timeout 300 python tools/solve_bench.py c1 > gpurun_out/c1_full_c.log 2>&1
grep -E "passed|failed|rc=" gpurun_out/t15.log | tail -3; cat gpurun_out/c5_full_c.log gpurun_out/c4_full_c.log gpurun_out/c3_full_c.log gpurun_out/c1_full_c.log
