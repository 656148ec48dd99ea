# session 3: paired-chunk epilogue of the fp16 tcgen05 kernel: parity on the tc tests, timing sweep
CNTGW_TC_PAIR=1 CNTGW_TC_POLY=3 timeout 900 python -m pytest tests/test_gpu_softmin.py tests/test_gpu_dist.py -q -m gpu -p no:cacheprovider -x -k "low_rank or c2 or tc or partial" > gpurun_out/s3_pair_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s3_pair_tests.log
timeout 600 python tools/sweep_paths.py 1048576 5 "C2 K=16 prec=2" > gpurun_out/s3_sweep_pair.log 2>&1; cat gpurun_out/s3_sweep_pair.log
