# session 3: full GPU suite, smoke, default bench line, reference arm, torchrun single-rank bench, launch list of the bench
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_48_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/s3_48_smoke.log
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/s3_48_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s3_48_tests.log | cut -c1-300
timeout 1200 python bench.py > gpurun_out/s3_48_bench.log 2>&1; echo "bench rc=$?"; tail -c 600 gpurun_out/s3_48_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/s3_48_bench_ref.log 2>&1; echo "ref rc=$?"; tail -c 400 gpurun_out/s3_48_bench_ref.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --no-solve > gpurun_out/s3_48_bench_torchrun.log 2>&1; echo "torchrun rc=$?"; tail -c 300 gpurun_out/s3_48_bench_torchrun.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2_bench_launches_f16.csv python bench.py --steps 2 --warmup 3 --no-solve --no-cpu-baseline --no-e2e > gpurun_out/s3_48_ncu.log 2>&1; echo "ncu rc=$?"
