# quick GPU iteration: tests ($TESTS) + per-workload bench lines ($WLS)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_umma.py} -x -q 2>&1 | tail -15 > gpurun_out/pytest_quick.log
cat gpurun_out/pytest_quick.log
for w in ${WLS:-cora pubmed}; do
  timeout 600 python bench.py --steps 200 --warmup 3 --no-cpu-baseline --workload $w > gpurun_out/qb_$w.json 2> gpurun_out/qb_$w.err
  python - "$w" <<'P'
import json,sys
w=sys.argv[1]
try:
    d=json.loads(open(f'gpurun_out/qb_{w}.json').read().strip().splitlines()[-1])
except Exception as e:
    print(w, 'FAILED', e); print(open(f'gpurun_out/qb_{w}.err').read()[-2000:]); sys.exit()
print(w, 'value', d['value'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'])
for k in d['kernels']: print(f"   {k['label']:40s} {k['ms']:.4f} {k['gb_s']}")
P
done
