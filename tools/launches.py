import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr=None; data=[]
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
names=[d['Kernel Name'] for d in data]
idx=[i for i,n in enumerate(names) if 'at::' in n and 'fill' in n.lower()]
step=data[idx[-1]+1:]
agg=collections.defaultdict(lambda:[0,0.0])
for d in step:
    n=d['Kernel Name'].split('(')[0][-40:]; v=float(d['Metric Value'])
    agg[n][0]+=1; agg[n][1]+=v
tot=sum(v[1] for v in agg.values())
print('step kernels', len(step), 'sum of kernel times (ms)', round(tot/1e6,3))
for n,(c,t) in sorted(agg.items(), key=lambda x:-x[1][1]):
    print(f"{t/1e3:10.1f} us {100*t/tot:5.1f}% {c:4d}  {n}")
if len(sys.argv)>2:
    for k in sys.argv[2:]:
        print(k, [ (d['Grid Size'].split(',')[0][1:], round(float(d['Metric Value'])/1e3,1)) for d in step if k in d['Kernel Name']])
