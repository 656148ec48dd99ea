# session 3: launch list of the probe sweeps (C4 and C5 laws), ncu --set full of the tcgen05 probe (summary only)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file /tmp/probe_c4.csv python tools/f64s_trace.py 1048576 0 2 c4 > gpurun_out/s3_13_a.log 2>&1; echo "rc=$?"
python /dev/stdin /tmp/probe_c4.csv > gpurun_out/s3_13_probe_c4_launches.txt <<'P'
import csv,sys,re
rows=list(csv.reader(open(sys.argv[1])))
hdr=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]
h=rows[hdr]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
for r in rows[hdr+1:]:
    if len(r)>vi:
        try: v=float(r[vi].replace(',',''))
        except: continue
        if v>20000: print(f"{v/1e6:9.3f} ms  {re.sub(r'\(.*','',r[ki])[:90]}")
P
head -60 gpurun_out/s3_13_probe_c4_launches.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:f64s_tcp_kernel --launch-skip 0 --launch-count 1 -o /tmp/r2_ncu_tcp_c4 python tools/f64s_trace.py 1048576 0 1 c4 > gpurun_out/s3_13_b.log 2>&1; echo "rc=$?"
python tools/ncu_summary.py /tmp/r2_ncu_tcp_c4.ncu-rep > gpurun_out/r2_ncu_tcprobe_c4.txt 2>&1; python tools/ncu_hot.py /tmp/r2_ncu_tcp_c4.ncu-rep 2>/dev/null | head -30 >> gpurun_out/r2_ncu_tcprobe_c4.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:f64s_tcp_kernel --launch-skip 0 --launch-count 1 -o /tmp/r2_ncu_tcp_c5 python tools/f64s_trace.py 262144 0 1 c5 > gpurun_out/s3_13_c.log 2>&1; echo "rc=$?"
python tools/ncu_summary.py /tmp/r2_ncu_tcp_c5.ncu-rep > gpurun_out/r2_ncu_tcprobe_c5.txt 2>&1; python tools/ncu_hot.py /tmp/r2_ncu_tcp_c5.ncu-rep 2>/dev/null | head -30 >> gpurun_out/r2_ncu_tcprobe_c5.txt
cat gpurun_out/r2_ncu_tcprobe_c4.txt gpurun_out/r2_ncu_tcprobe_c5.txt
