python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/repro_f32c.py 5 > gpurun_out/rep2.log 2>&1; echo rc=$? >> gpurun_out/rep2.log
timeout 1200 python tools/f64s_trace.py 262144 1 60 > gpurun_out/f64s_trace.log 2>&1
tail -n 3 gpurun_out/rep2.log; cat gpurun_out/f64s_trace.log | tail -62
