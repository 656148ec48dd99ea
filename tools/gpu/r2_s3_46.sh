# session 3: F64S from 2^27 pairs (kd < 16) / 2^24 pairs (kd >= 16): full GPU suite, mid-size solves, bench solve block
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/s3_46_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s3_46_tests.log | cut -c1-300
for cfg in "c4 65536 5" "c5 32768 5" "c4 16384 4" "c5 4096 4" "c3"; do
  timeout 300 python tools/solve_bench.py $cfg > /tmp/a.log 2>&1; python -c "
import json; d=json.loads(open('/tmp/a.log').read().strip().splitlines()[-1]); print('$cfg', 'path', d.get('precision_path'), round(d['seconds'],3), d.get('step_seconds'), (d.get('objectives') or d.get('stage_values'))[-1])"
done 2>&1 | tee gpurun_out/s3_46_mid.log
