import csv,sys,collections
def fl(x):
    try: return float(x)
    except: return 0.0
rows=list(csv.reader(open(sys.argv[1])))
secs=[];cur=None;name=None
for r in rows:
    if r and r[0] in ("Function Name","Kernel Name"): name=r[1]; continue
    if r and r[0]=="Address": cur={'name':name,'hdr':r,'rows':[]}; secs.append(cur); continue
    if cur is not None and r and r[0] not in("File Path",): cur['rows'].append(r)
for s in secs:
    h=s['hdr']; ia=h.index("Warp Stall Sampling (All Samples)"); isrc=h.index("Source"); iex=h.index("Instructions Executed")
    sc=[i for i,c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    tot=sum(fl(r[ia]) for r in s['rows'])
    print("====",s['name'][:110],"samples",tot)
    seg=collections.Counter(); segn=0; segi=0; kinds=collections.Counter(); first=None
    def flush(lbl):
        global seg,segn,segi,kinds,first
        if segn:
            top=dict(sorted(seg.items(),key=lambda kv:-kv[1])[:5])
            print(f"  seg {first:>6} n={segn:4d} exec={segi/1e6:8.1f}M samples={sum(seg.values())/tot*100:5.1f}% {({k:round(v/tot*100,1) for k,v in top.items()})} {dict(kinds.most_common(6))} -> {lbl}")
        seg=collections.Counter(); segn=0; segi=0; kinds=collections.Counter(); first=None
    for r in s['rows']:
        if len(r)<=ia: continue
        ins=r[isrc].strip()
        if first is None: first=r[0][-5:]
        op=ins.split()[0] if not ins.startswith('@') else ins.split()[1]
        kinds[op.split('.')[0]]+=1
        for i in sc: seg[h[i][6:]]+=fl(r[i])
        segn+=1; segi+=fl(r[iex])
        if op.startswith("BAR") or op.startswith("EXIT"): flush(ins[:40])
    flush("end")
