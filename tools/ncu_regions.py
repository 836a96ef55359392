import csv, io, subprocess, sys, collections, re
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","cuda,sass","--kernel-name","regex:"+kern,"-c","1"],capture_output=True,text=True).stdout
fname=""; rows=[]; hdr=None
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0]=="File Path": fname=r[1].split("/")[-1]; continue
    if r[0]=="Line No": hdr=r; continue
    try: ln=int(r[0])
    except: continue
    try:
        rows.append((fname,ln,float(r[7]),float(r[4]),r[1].strip()[:80]))
    except (ValueError, IndexError):
        continue
print(hdr)
tot=sum(x[2] for x in rows); tots=sum(x[3] for x in rows)
print("total inst",tot, "samples", tots)
# ranges: file -> list of (lo,hi,name)
R=eval(open(sys.argv[3]).read()) if len(sys.argv)>3 else {}
agg=collections.OrderedDict()
for f,ln,i,s,src in rows:
    name=f
    for lo,hi,nm in R.get(f,[]):
        if lo<=ln<=hi: name=f+":"+nm; break
    a=agg.setdefault(name,[0,0]); a[0]+=i; a[1]+=s
for k,(i,s) in sorted(agg.items(), key=lambda kv:-kv[1][0]):
    print(f"{100*i/tot:5.1f}% inst {100*s/max(tots,1):5.1f}% stall  {k}")
