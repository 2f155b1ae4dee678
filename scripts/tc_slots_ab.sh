# k_fbb_tc piece rows x ring slots on products (per-op time of the paired FBB and the forward)
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for cfg in "128 4" "64 8" "64 6" "32 8" "128 2"; do
  set -- $cfg
  echo "pr=$1 slots=$2 $(BG_TC_PR=$1 BG_TC_SLOTS=$2 python bench.py --workload products --steps 20 --warmup 5 --no-cpu-baseline --no-clocks 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], [k["ms"] for k in d["kernels"] if "pair" in k["label"]])')"
done
done
