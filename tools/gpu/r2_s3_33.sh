timeout 300 python tools/k4_density.py c4 1048576 3 > gpurun_out/s3_33_k4.log 2>&1; cat gpurun_out/s3_33_k4.log | tail -5
timeout 300 python tools/k4_density.py c5 262144 3 >> gpurun_out/s3_33_k4.log 2>&1; cat gpurun_out/s3_33_k4.log | tail -4
