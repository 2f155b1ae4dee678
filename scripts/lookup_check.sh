# packed FBF lookup: model-level parity (sage / saint, paired and not) and the products forward
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_pair.py tests/test_gpu_layers.py tests/test_gpu_glue_layers.py tests/test_gpu_edge_cases.py -x -q -m gpu 2>&1 | tail -1
python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu -k "product" 2>&1 | tail -1
for rep in 1 2; do
  echo "$(python bench.py --workload products --steps 20 --warmup 5 --no-cpu-baseline --no-clocks 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], [(k["label"], k["ms"]) for k in d["kernels"] if "FBF" in k["label"]])')"
done
NCU_K="k_fbf_lookup" NCU_SKIP=3 WL=products NAME=s3_lookup2 bash scripts/ncu_one.sh 2>&1 | grep -E "duration|dram write|instructions|issue"
