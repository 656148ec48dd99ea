python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in "" "CNTGW_K4_SPARSE=0" "CNTGW_CTR_SKIP=0" "CNTGW_CTR_REUSE=0" "CNTGW_K4_SPARSE=0 CNTGW_CTR_SKIP=0"; do
  echo "== $v" >> gpurun_out/rep.log
  env $v CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/repro_f32c.py 5 >> gpurun_out/rep.log 2>&1
  echo "rc=$?" >> gpurun_out/rep.log
done
grep -E "==|rc=|Error|error|^[0-9]" gpurun_out/rep.log | head -40
