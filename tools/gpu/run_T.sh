python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for T in 48 40; do CNTGW_CTR_SKIP_T=$T timeout 600 python tools/ctr_check.py half c4 1048576 100 > gpurun_out/half_T$T.log 2>&1; done
