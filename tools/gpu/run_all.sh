python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench.log 2>&1
timeout 900 python tools/solve_bench.py c3 > gpurun_out/solve_c3.log 2>&1
timeout 300 python tools/solve_bench.py c1 > gpurun_out/solve_c1.log 2>&1
tail -n 2 gpurun_out/gpu_tests.log gpurun_out/smoke.log
