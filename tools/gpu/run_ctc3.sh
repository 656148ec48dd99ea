python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_softmin.py -x -q -k "f32c or centred" > gpurun_out/t_ctc3.log 2>&1
timeout 300 python tools/ctr_check.py half c4 1048576 5 > gpurun_out/half_ctc3.log 2>&1
timeout 1200 python tools/ctr_check.py c4 1048576 3 100 > gpurun_out/ctr_c4_3step_tc3.log 2>&1
tail -n 3 gpurun_out/t_ctc3.log
