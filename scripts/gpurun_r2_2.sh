cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_tileset.py tests/test_gpu_layers.py tests/test_gpu_container.py tests/test_cpp_shim.py -x -q > gpurun_out/r2_t2.log 2>&1
echo "rc=$?" >> gpurun_out/r2_t2.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "digests" >> gpurun_out/r2_t2.log 2>&1
echo "rc=$?" >> gpurun_out/r2_t2.log
tail -5 gpurun_out/r2_t2.log
