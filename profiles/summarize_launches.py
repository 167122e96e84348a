import csv, collections, sys
def summarize(path, top=25):
    rows=list(csv.reader(open(path)))
    hdr=None; data=[]
    for r in rows:
        if r and r[0]=='ID': hdr=r; continue
        if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
    agg=collections.defaultdict(lambda:[0,0.0])
    for d in data:
        name=d['Kernel Name'].split('(')[0][:60]; v=float(d['Metric Value'])
        agg[name][0]+=1; agg[name][1]+=v
    tot=sum(v[1] for v in agg.values())
    print('launches',len(data),'total us',tot/1e3)
    for k,(n,v) in sorted(agg.items(), key=lambda x:-x[1][1])[:top]: print(f"{k:60s} {n:5d} {v/1e3:10.1f} us  avg {v/1e3/n:8.1f} us {100*v/tot:5.1f}%")
if __name__=="__main__":
    import signal; signal.signal(signal.SIGPIPE, signal.SIG_DFL); summarize(sys.argv[1])
