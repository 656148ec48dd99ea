python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for P in 2 4 0; do CNTGW_TC_POLY=$P python bench.py --steps 6 --warmup 3 > gpurun_out/bench_poly$P.log 2>&1; done
