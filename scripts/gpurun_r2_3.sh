cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_layers.py tests/test_gpu_verify.py tests/test_cpp_shim.py tests/test_gpu_parity.py -x -q > gpurun_out/r2_t3.log 2>&1
echo "rc=$?" >> gpurun_out/r2_t3.log
tail -5 gpurun_out/r2_t3.log
