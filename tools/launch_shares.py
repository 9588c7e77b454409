import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hdr]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
agg=collections.defaultdict(lambda:[0,0.0])
for r in rows[hdr+1:]:
    try: v=float(r[vi].replace(',',''))
    except: continue
    if r[ui]=='usecond': v*=1e3
    if r[ui]=='msecond': v*=1e6
    agg[r[ki][:80]][0]+=1; agg[r[ki][:80]][1]+=v
tot=sum(v[1] for v in agg.values())
for k,v in sorted(agg.items(), key=lambda x:-x[1][1]): print(f"{v[0]:5d} {v[1]/1e3:11.1f}us {100*v[1]/tot:5.1f}%  {k}")
