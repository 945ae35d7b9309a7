"""Per-source-line share of warp-stall samples and executed instructions from an ncu --set full
report captured with --import-source on:
    ncu -i REP --page source --csv --print-source cuda,sass > SRC.csv; python profiles/hotlines.py SRC.csv [N]
"""
import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
f=None; agg={}
for r in rows:
    if len(r)==2 and r[0]=='File Path': f=r[1].split('/')[-1]; continue
    if len(r)<8 or r[0] in ('Line No','Function Name'): continue
    if r[0].isdigit():
        try: samp=int(r[4] or 0); ins=int(r[7] or 0)
        except: samp=ins=0
        agg[(f,int(r[0]),r[1].strip()[:80])]=(samp,ins)
tot=sum(v[0] for v in agg.values()) or 1; ti=sum(v[1] for v in agg.values()) or 1
print("total samples",tot,"inst",ti)
for k,v in sorted(agg.items(), key=lambda kv:-kv[1][0])[:int(sys.argv[2]) if len(sys.argv)>2 else 40]:
    print(f"{v[0]/tot*100:5.1f}% {v[1]/ti*100:5.1f}%  {k[0]}:{k[1]}  {k[2]}")
