cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_persistent.py -x -q > gpurun_out/r2_t6.log 2>&1
echo "rc=$?" >> gpurun_out/r2_t6.log
tail -15 gpurun_out/r2_t6.log
WL=cora bash scripts/quick_bench.sh
WL=pubmed bash scripts/quick_bench.sh
