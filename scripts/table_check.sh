# packed FBF softmax table (warp per row): model-level parity and the products / Flickr forwards
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_pair.py tests/test_gpu_layers.py tests/test_gpu_glue_layers.py tests/test_gpu_edge_cases.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1
python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu -k "product or flickr" 2>&1 | tail -1
for wl in products flickr; do for rep in 1 2; do
  echo "$wl $(python bench.py --workload $wl --steps 30 --warmup 5 --no-cpu-baseline --no-clocks 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], [(k["label"], k["ms"]) for k in d["kernels"] if "FBF" in k["label"]])')"
done; done
WLS="products flickr" NCU_CACHE=none bash scripts/launches.sh 2>&1 | grep -E "fbf_table" | head -4
