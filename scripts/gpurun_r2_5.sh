cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_glue_layers.py tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_sharded.py tests/test_gpu_layers.py -x -q > gpurun_out/r2_t5.log 2>&1
echo "rc=$?" >> gpurun_out/r2_t5.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "products" >> gpurun_out/r2_t5.log 2>&1
echo "rc=$?" >> gpurun_out/r2_t5.log
tail -4 gpurun_out/r2_t5.log
WL=products bash scripts/quick_bench.sh
