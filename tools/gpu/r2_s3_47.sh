# session 3: C3 chain A/B: F64S threshold 2^27 (new default) vs 2^34 (old), 3 runs each, interleaved
for rep in 1 2 3; do for mp in default 17179869184; do
  if [ $mp = default ]; then unset CNTGW_F64S_MIN_PAIRS; else export CNTGW_F64S_MIN_PAIRS=$mp; fi
  timeout 300 python tools/solve_bench.py c3 > /tmp/a.log 2>&1; python -c "
import json; d=json.loads(open('/tmp/a.log').read().strip().splitlines()[-1]); print('c3 min_pairs=$mp', round(d['seconds'],3), d['stage_values'][-1], d['error'])"
done; done 2>&1 | tee gpurun_out/s3_47_c3.log
