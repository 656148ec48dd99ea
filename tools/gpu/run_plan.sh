python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_softmin.py -x -q -k "f32c or centred or zero_weight" > gpurun_out/t_plan.log 2>&1
timeout 600 python tools/ctr_check.py half c4 1048576 100 > gpurun_out/half_plan_100.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ctr_plan|softmin_ctr_kernel" --csv --log-file gpurun_out/launches_plan.csv python tools/ctr_check.py half c4 1048576 5 > gpurun_out/ncu_launch_plan.log 2>&1
tail -n 2 gpurun_out/t_plan.log
