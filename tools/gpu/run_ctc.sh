python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_softmin.py -x -q -k "f32c or centred" > gpurun_out/t_ctc.log 2>&1
for P in 4; do
CNTGW_CTR_TC_POLY=$P timeout 300 python tools/ctr_check.py half c4 1048576 5 > gpurun_out/half_ctc_p$P.log 2>&1
done
tail -n 3 gpurun_out/t_ctc.log
