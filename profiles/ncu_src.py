import csv, sys, subprocess, collections
rep=sys.argv[1]; topn=int(sys.argv[2]) if len(sys.argv)>2 else 40
out=subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source=cuda,sass"],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
agg=collections.defaultdict(lambda:[0,0,''])
cur=None; hdr=None
for r in rows:
    if not r: continue
    if r[0]=='File Path': cur=r[1].split('/')[-1]; continue
    if r[0]=='Function Name': continue
    if r[0]=='Line No': hdr=r; continue
    if hdr is None: continue
    d=dict(zip(hdr,r))
    try: line=int(r[0])
    except: continue
    try:
        agg[(cur,line)][0]+=float(d.get('Instructions Executed','0') or 0); agg[(cur,line)][1]+=float(d.get('Warp Stall Sampling (All Samples)','0') or 0); agg[(cur,line)][2]=r[1][:100]
    except: pass
ti=sum(v[0] for v in agg.values()); ts=sum(v[1] for v in agg.values())
print('total inst %.3e samples %.3e'%(ti,ts))
for k,v in sorted(agg.items(), key=lambda kv:-kv[1][1])[:topn]:
    print(f"{k[0][:14]:14s}:{k[1]:4d} inst {100*v[0]/ti:5.1f}% stall {100*v[1]/ts:5.1f}%  {v[2]}")
