# round 2, trip 4: K4 same-pair test, C3 chain diagnosis, precision bound, C5 sparsity probe
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_integration.py -q -s -m gpu -p no:cacheprovider > gpurun_out/t7.log 2>&1; echo rc=$? >> gpurun_out/t7.log
timeout 300 python tools/c3_chain_diag.py > gpurun_out/c3diag.log 2>&1
CNTGW_DEVICE_LOOP=0 timeout 300 python tools/c3_chain_diag.py > gpurun_out/c3diag_host.log 2>&1
timeout 1500 python tools/c5_sparsity.py 262144 2 50 > gpurun_out/c5sparsity.log 2>&1
tail -n 3 gpurun_out/t7.log
