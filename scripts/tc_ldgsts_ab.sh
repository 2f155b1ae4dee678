# k_fbb_tc: bulk-copy producer vs 32-lane cp.async producer (products), parity under both
cd $GRAFT_REPO_ROOT
BG_TC_LDGSTS=1 python -m pytest tests/test_gpu_pair.py tests/test_gpu_umma.py -x -q -m gpu -k "tc or default" 2>&1 | tail -1
for rep in 1 2; do
for cfg in "0 4" "1 4" "1 3" "1 2"; do
  set -- $cfg
  echo "ldgsts=$1 slots=$2 $(BG_TC_LDGSTS=$1 BG_TC_SLOTS=$2 python bench.py --workload products --steps 20 --warmup 5 --no-cpu-baseline --no-clocks 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], [k["ms"] for k in d["kernels"] if "pair" in k["label"]])')"
done
done
