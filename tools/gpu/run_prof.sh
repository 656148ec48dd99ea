python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:softmin_ctr_kernel -c 1 -o gpurun_out/ncu_ctr_final python tools/ctr_check.py half c4 1048576 5 > gpurun_out/ncu_ctr_final.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c4_half.csv python tools/ctr_check.py half c4 1048576 2 > gpurun_out/ncu_launch.log 2>&1
ls -la gpurun_out | tail -5
