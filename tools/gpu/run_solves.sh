python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python tools/solve_bench.py c4 > gpurun_out/solve_c4.log 2>&1
timeout 1500 python tools/solve_bench.py c5 > gpurun_out/solve_c5.log 2>&1
timeout 300 python tools/solve_bench.py c1 > gpurun_out/solve_c1.log 2>&1
timeout 300 python tools/solve_bench.py c3 > gpurun_out/solve_c3.log 2>&1
