python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python tools/solve_bench.py c3 > gpurun_out/solve_c3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"softmin_ctr_kernel|ctr_plan" -c 2 -o gpurun_out/ncu_ctr_r4 python tools/ctr_check.py half c4 1048576 100 > gpurun_out/ncu_ctr_r4.log 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_c4.txt
timeout 3000 python tools/ctr_check.py c4 1048576 10 100 > gpurun_out/ctr_c4_1m_final.log 2>&1
tail -n 2 gpurun_out/ctr_c4_1m_final.log
