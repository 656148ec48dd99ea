python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_softmin.py -x -q -k "f32c or centred" > gpurun_out/t_ctc.log 2>&1
timeout 300 python tools/ctr_check.py half c4 1048576 5 > gpurun_out/half_ctc_p4.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:softmin_ctc -c 1 -o gpurun_out/ncu_ctc_c4_v3 python tools/ctr_check.py half c4 1048576 5 > gpurun_out/ncu_ctc.log 2>&1
tail -n 3 gpurun_out/t_ctc.log
