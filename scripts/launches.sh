# per-kernel durations (ncu launch list) of one small-workload bench run: WL=cora|pubmed|...
cd $GRAFT_REPO_ROOT
for w in ${WLS:-cora pubmed}; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control ${NCU_CACHE:-all} --csv --log-file gpurun_out/launch_$w.csv python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline --no-clocks > /dev/null 2>&1
python - $w <<'P'
import csv,sys,collections
w=sys.argv[1]
rows=[r for r in csv.reader(open(f'gpurun_out/launch_{w}.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ii=h.index('ID')
ks=[(int(r[ii]),r[ki],float(r[vi])) for r in rows[1:]]
print(w, len(ks), 'launches')
for i,k,v in ks[-16:]: print(f'  {i:5d} {v/1000 if v>1000 else v:9.2f} {k[:90]}')
P
done
