python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_native_solve.py tests/test_gpu_dist.py -q -s -m gpu -p no:cacheprovider > gpurun_out/t18.log 2>&1; echo rc=$? >> gpurun_out/t18.log
tail -n 25 gpurun_out/t18.log
