import csv,sys,subprocess
rep=sys.argv[1]; top=int(sys.argv[2]) if len(sys.argv)>2 else 45
txt=subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","cuda,sass"],capture_output=True,text=True).stdout
rows=list(csv.reader(txt.splitlines()))
cur=None; out=[]; tot=0
for r in rows:
    if len(r)>=2 and r[0]=='File Path': cur=r[1].split('/')[-1]; continue
    if len(r)>7 and r[0].isdigit():
        out.append((int(r[7]) if r[7].isdigit() else 0, int(r[6]) if r[6].isdigit() else 0, cur, int(r[0]), r[1].strip()[:120]))
    elif len(r)>7 and r[0]=='' and r[7].isdigit(): tot+=int(r[7])
print("total warp inst",tot)
out.sort(reverse=True); s=0
for ie,sm,f,ln,src in out[:top]:
    s+=ie; print(f"{100*ie/tot:5.2f}% cum {100*s/tot:5.1f}% smp {sm:7d} {f}:{ln}  {src}")
