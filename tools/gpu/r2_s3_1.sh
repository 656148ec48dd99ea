# session-3 re-entry check: full GPU suite, default bench line, C4/C5 solve step times on the probe-measured F64S path
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/s3_1_smi.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/s3_1_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/s3_1_tests.log
timeout 1200 python bench.py > gpurun_out/s3_1_bench.log 2>&1; echo "bench rc=$?"; tail -c 4000 gpurun_out/s3_1_bench.log
