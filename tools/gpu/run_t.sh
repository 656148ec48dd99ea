python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_softmin.py tests/test_gpu_dist.py -x -q > gpurun_out/t_sm.log 2>&1
tail -n 3 gpurun_out/t_sm.log
