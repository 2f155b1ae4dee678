# one bench line without the CPU baseline; per-kernel table to stdout
cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 100 --warmup 3 --no-cpu-baseline ${WL:+--workload $WL} > gpurun_out/qb.json 2> gpurun_out/qb.err
python - <<'P'
import json
d=json.loads(open('gpurun_out/qb.json').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'])
for k in d['kernels']: print(f"{k['label']:40s} {k['ms']:.4f} {k['gb_s']}")
P
