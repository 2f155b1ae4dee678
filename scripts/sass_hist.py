"""Per-opcode instruction and stall-sample histogram of an ncu source-page CSV
(ncu -i X.ncu-rep --page source --csv --print-source sass > X.csv).
usage: sass_hist.py X.csv"""
import csv,sys,collections
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[1]; data=rows[2:]
ia=hdr.index("Instructions Executed"); isrc=hdr.index("Source"); iss=hdr.index("Warp Stall Sampling (All Samples)")
tot=0; byop=collections.Counter(); st=collections.Counter(); stall_tot=0
for r in data:
    n=int(r[ia] or 0); s=r[isrc].strip()
    op=s.split()[0] if s else '?'
    if op.startswith('@'): op=s.split()[1]
    op=op.split('.')[0]
    byop[op]+=n; tot+=n
    st[op]+=int(r[iss] or 0); stall_tot+=int(r[iss] or 0)
print('total warp inst',tot)
for op,n in byop.most_common(25): print(f'{op:12s} {n:12d} {n/tot*100:5.1f}%  stall-samples {st[op]/stall_tot*100:5.1f}%')
# top lines by stall samples
print('--- top lines by samples')
top=sorted(data,key=lambda r:-int(r[iss] or 0))[:25]
for r in top: print(r[0][-5:], r[isrc].strip()[:60], r[iss], r[ia])
