# session 3: fp16-operand tcgen05 kernel as the default: full GPU suite, bench, ncu of the bench kernel (summary only)
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/s3_6_tests.log 2>&1; echo "tests rc=$?"; tail -6 gpurun_out/s3_6_tests.log
timeout 1200 python bench.py > gpurun_out/s3_6_bench.log 2>&1; echo "bench rc=$?"; tail -c 2500 gpurun_out/s3_6_bench.log | head -c 1800
timeout 900 ncu --set full --import-source on --clock-control none -k regex:softmin_tc_kernel --launch-skip 4 --launch-count 1 -o /tmp/r2_ncu_tc_f16 python bench.py --steps 2 --warmup 3 --no-solve --no-cpu-baseline --no-e2e > gpurun_out/s3_6_ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py /tmp/r2_ncu_tc_f16.ncu-rep > gpurun_out/r2_ncu_tc_f16_c2.txt 2>&1
python tools/ncu_summary.py --traffic-json gpurun_out/r2_bench_traffic.json /tmp/r2_ncu_tc_f16.ncu-rep 1048576 1048576 >> gpurun_out/s3_6_ncu.log 2>&1
python tools/ncu_hot.py /tmp/r2_ncu_tc_f16.ncu-rep 2>/dev/null | head -40 >> gpurun_out/r2_ncu_tc_f16_c2.txt
cat gpurun_out/r2_ncu_tc_f16_c2.txt | head -40
