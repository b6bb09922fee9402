import csv,collections,sys
rows=list(csv.reader(open(sys.argv[1])))
n_inf=int(sys.argv[2]) if len(sys.argv)>2 else 4
hdr=None;agg=collections.defaultdict(lambda:[0,0.0])
for r in rows:
    if len(r)>10 and r[0]=='ID': hdr=r;continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d['Metric Name']=='gpu__time_duration.sum':
            k=d['Kernel Name'][:60]; agg[k][0]+=1; agg[k][1]+=float(d['Metric Value'])/1e6
for k,v in sorted(agg.items(),key=lambda x:-x[1][1]): print(f"{v[1]/n_inf:9.2f} ms/inf {v[0]/n_inf:6.1f} {k}")
