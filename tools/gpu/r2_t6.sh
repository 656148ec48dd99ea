python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1800 python tools/c5_drift.py 262144 1 > gpurun_out/c5drift.log 2>&1
tail -n 20 gpurun_out/c5drift.log
