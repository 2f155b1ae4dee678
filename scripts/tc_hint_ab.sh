# products bench under several try_wait suspend hints for k_fbb_tc, plus the tc parity tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m pytest tests/test_gpu_pair.py tests/test_gpu_umma.py -x -q -m gpu -k "tc or default" 2>&1 | tail -2
for rep in 1 2; do
  for h in 0 2000 20000 1000000; do
    echo "hint=$h $(BG_TC_HINT=$h python bench.py --workload products --steps 20 --warmup 5 --no-cpu-baseline --no-clocks 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"])')"
  done
done
