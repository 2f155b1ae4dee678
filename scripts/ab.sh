# A/B: one bench per env setting (ENVS="A=1 B=2;C=3" separated by ';'), kernels table each
cd $GRAFT_REPO_ROOT
IFS=';' read -ra SETS <<< "${ENVS:-}"
[ ${#SETS[@]} -eq 0 ] && SETS=("")
i=0
for e in "${SETS[@]}"; do
  env $e timeout 600 python bench.py --steps 100 --warmup 3 --no-cpu-baseline ${WL:+--workload $WL} > gpurun_out/ab$i.json 2> gpurun_out/ab$i.err
  echo "== [$e]"
  python - $i <<'P'
import json,sys
i=sys.argv[1]
try:
  d=json.loads(open(f'gpurun_out/ab{i}.json').read().strip().splitlines()[-1])
except Exception as ex:
  print('FAILED', ex); print(open(f'gpurun_out/ab{i}.err').read()[-1500:]); sys.exit()
print('value', d['value'], 'frac', d['roofline']['frac'], 'bbfrac', d.get('roofline_bit_spmm',{}).get('frac'), 'maxdiff', d.get('output_max_abs_diff'))
for k in d['kernels']: print(f"  {k['label']:40s} {k['ms']:.4f} {k['gb_s']}")
P
  i=$((i+1))
done
