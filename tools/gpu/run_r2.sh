python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CNTGW_CTR_R=2 timeout 300 python -m pytest tests/test_gpu_softmin.py -x -q -k "f32c or centred or zero_weight" > gpurun_out/t_r2.log 2>&1
CNTGW_CTR_R=2 timeout 600 python tools/ctr_check.py half c4 1048576 100 > gpurun_out/half_r2_100.log 2>&1
CNTGW_CTR_R=2 timeout 600 python tools/ctr_check.py half c4 1048576 5 > gpurun_out/half_r2_5.log 2>&1
timeout 600 python tools/ctr_check.py half c4 1048576 5 > gpurun_out/half_r4_5b.log 2>&1
tail -n 1 gpurun_out/t_r2.log
