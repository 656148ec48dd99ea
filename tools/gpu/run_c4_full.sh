python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_c4.txt
timeout 3000 python tools/ctr_check.py c4 1048576 10 100 > gpurun_out/ctr_c4_1m_full_skip_r4.log 2>&1
tail -n 2 gpurun_out/ctr_c4_1m_full_skip_r4.log
