# round 2, trip 1: new parity tests + short bench
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu --ignore=tests/test_gpu_fullsize.py -p no:cacheprovider > gpurun_out/t1.log 2>&1; echo rc=$? >> gpurun_out/t1.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -s -m gpu -p no:cacheprovider > gpurun_out/t2.log 2>&1; echo rc=$? >> gpurun_out/t2.log
timeout 900 python bench.py --steps 3 --warmup 3 --size 262144 --solve-n 262144 --solve-outer 2 > gpurun_out/b1.log 2>&1; echo rc=$? >> gpurun_out/b1.log
tail -n 3 gpurun_out/t1.log gpurun_out/t2.log gpurun_out/b1.log
