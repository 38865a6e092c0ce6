import csv,sys,collections
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[1]; data=rows[2:]
ix={h:i for i,h in enumerate(hdr)}
tot=0; by=collections.Counter(); samp=collections.Counter(); thr=collections.Counter()
recs=[]
for r in data:
    if len(r)<len(hdr): continue
    src=r[ix['Source']].strip(); op=src.split()[0] if src else ''
    if op.startswith('@'): op=src.split()[1]
    opb=op.split('.')[0]
    n=int(r[ix['Instructions Executed']] or 0); s=int(r[ix['Warp Stall Sampling (All Samples)']] or 0)
    t=int(r[ix['Thread Instructions Executed']] or 0)
    tot+=n; by[opb]+=n; samp[opb]+=s; thr[opb]+=t
    recs.append((s,n,r[ix['Address']][-5:],src))
print('total warp inst',tot, 'samples', sum(samp.values()))
for k,v in by.most_common(30): print(f'{k:10s} {v/tot*100:5.1f}% inst  {samp[k]/sum(samp.values())*100:5.1f}% samples  thr/inst {thr[k]/max(v,1):.1f}')
recs.sort(reverse=True)
for s,n,a,src in recs[:40]: print(s,n,a,src)
