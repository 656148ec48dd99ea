python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_softmin.py tests/test_gpu_solver.py tests/test_gpu_dist.py -x -q > gpurun_out/t_reuse.log 2>&1
tail -n 2 gpurun_out/t_reuse.log
timeout 2400 python tools/ctr_check.py c4 1048576 10 100 > gpurun_out/ctr_c4_1m_reuse.log 2>&1
tail -n 1 gpurun_out/ctr_c4_1m_reuse.log | cut -c1-400
