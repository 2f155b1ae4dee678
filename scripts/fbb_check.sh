# FBB kernels: parity tests, then products / Flickr / Reddit bench ms
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m pytest tests/test_gpu_pair.py tests/test_gpu_umma.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for wl in ${WLS:-products flickr reddit}; do
  for rep in 1 2; do
    echo "$wl $(python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline --no-clocks 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], d.get("roofline",{}).get("frac"))')"
  done
done
