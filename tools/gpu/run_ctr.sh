python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_softmin.py -x -q -k "f32c or centred" -s > gpurun_out/t_ctr.log 2>&1
for L in 16384 65536 262144; do
CNTGW_CTR_TILE_LIMIT=$L timeout 600 python tools/ctr_check.py half c4 1048576 20 > gpurun_out/half_c4_1m_L$L.log 2>&1
done
tail -n 3 gpurun_out/t_ctr.log
