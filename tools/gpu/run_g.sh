python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CNTGW_CTR_G=8 timeout 600 python tools/ctr_check.py half c4 1048576 100 > gpurun_out/half_g8.log 2>&1
CNTGW_CTR_POLY=1 timeout 600 python tools/ctr_check.py half c4 1048576 100 > gpurun_out/half_p1.log 2>&1
