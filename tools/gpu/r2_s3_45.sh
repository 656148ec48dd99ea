# session 3: crossover of F64S against the dense fp64 path on the cold laws at small sizes
for n in 2048 4096 8192 16384; do for mp in 17179869184 1; do
  CNTGW_F64S_MIN_PAIRS=$mp timeout 300 python tools/solve_bench.py c4 $n 4 > /tmp/a.log 2>&1; python -c "
import json; d=json.loads(open('/tmp/a.log').read().strip().splitlines()[-1]); print('C4', $n, 'min_pairs=$mp', 'path', d['precision_path'], round(d['seconds'],3), d['step_seconds'], d['objectives'][-1])"
  CNTGW_F64S_MIN_PAIRS=$mp timeout 300 python tools/solve_bench.py c5 $n 4 > /tmp/a.log 2>&1; python -c "
import json; d=json.loads(open('/tmp/a.log').read().strip().splitlines()[-1]); print('C5', $n, 'min_pairs=$mp', 'path', d['precision_path'], round(d['seconds'],3), d['step_seconds'], d['objectives'][-1])"
done; done 2>&1 | tee gpurun_out/s3_45_crossover.log
