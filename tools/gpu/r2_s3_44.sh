# session 3: F64S size threshold: C3 (1e5) and mid sizes on F64S vs the dense fp64 path
for mp in 17179869184 1000000000; do
  CNTGW_F64S_MIN_PAIRS=$mp timeout 300 python tools/solve_bench.py c3 > gpurun_out/s3_44_c3_$mp.log 2>&1; tail -1 gpurun_out/s3_44_c3_$mp.log | cut -c1-400
done
for mp in 17179869184 1000000000; do
  CNTGW_F64S_MIN_PAIRS=$mp timeout 300 python tools/solve_bench.py c4 65536 5 > gpurun_out/s3_44_c4s_$mp.log 2>&1; tail -1 gpurun_out/s3_44_c4s_$mp.log | cut -c1-500
  CNTGW_F64S_MIN_PAIRS=$mp timeout 300 python tools/solve_bench.py c5 32768 5 > gpurun_out/s3_44_c5s_$mp.log 2>&1; tail -1 gpurun_out/s3_44_c5s_$mp.log | cut -c1-500
done
