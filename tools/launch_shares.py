"""Kernel shares of an `ncu --metrics gpu__time_duration.sum --csv` launch list.
Usage: python tools/launch_shares.py launches.csv [top_n]"""
import csv,collections,re,sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]
h=rows[hdr]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
agg=collections.defaultdict(lambda:[0,0.0])
for r in rows[hdr+1:]:
    if len(r)<=vi: continue
    try: v=float(r[vi].replace(',',''))
    except: continue
    k=re.sub(r'\(.*','',r[ki]); agg[k][0]+=1; agg[k][1]+=v
tot=sum(v[1] for v in agg.values())
for k,v in sorted(agg.items(), key=lambda kv:-kv[1][1])[:int(sys.argv[2]) if len(sys.argv)>2 else 22]: print(f"{v[1]/1e6:10.2f} ms {v[0]:6d} {100*v[1]/tot:5.1f}% {k[:110]}")
print('total ms',tot/1e6)
