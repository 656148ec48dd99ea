# session 3: F64S plan granularity sweep (rows per group x columns per stage) on the C5 and C4 solves
for cfg in "1 128" "2 64" "1 64"; do set -- $cfg
  CNTGW_F64S_RG=$1 CNTGW_F64S_TD=$2 timeout 600 python tools/solve_bench.py c5 262144 10 > gpurun_out/s3_21_c5_$1_$2.log 2>&1
  python -c "
import json,sys
d=json.loads(open('gpurun_out/s3_21_c5_$1_$2.log').read().strip().splitlines()[-1]); print('C5 rg=$1 td=$2', d['seconds'], d['step_seconds'], d['objectives'][-1])" 2>&1 | tail -1
done
for cfg in "1 256" "2 128" "1 128"; do set -- $cfg
  CNTGW_F64S_RG=$1 CNTGW_F64S_TD=$2 timeout 900 python tools/solve_bench.py c4 1048576 10 > gpurun_out/s3_21_c4_$1_$2.log 2>&1
  python -c "
import json,sys
d=json.loads(open('gpurun_out/s3_21_c4_$1_$2.log').read().strip().splitlines()[-1]); print('C4 rg=$1 td=$2', d['seconds'], d['step_seconds'], d['objectives'][-1])" 2>&1 | tail -1
done
