# session 3: where the C4-shape tcgen05 probe waits: ncu source-level stall samples with context
timeout 900 ncu --set full --import-source on --clock-control none -k regex:f64s_tcp_kernel --launch-skip 0 --launch-count 1 -o /tmp/r2_ncu_tcp_c4b python tools/f64s_trace.py 1048576 0 1 c4 > gpurun_out/s3_30_b.log 2>&1; echo "rc=$?"
python tools/ncu_summary.py /tmp/r2_ncu_tcp_c4b.ncu-rep > gpurun_out/r2_ncu_tcprobe_c4_ring16.txt 2>&1
python tools/ncu_hot.py /tmp/r2_ncu_tcp_c4b.ncu-rep 14 6 >> gpurun_out/r2_ncu_tcprobe_c4_ring16.txt 2>/dev/null
cat gpurun_out/r2_ncu_tcprobe_c4_ring16.txt
