cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu_full.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest_gpu_full.log
tail -3 gpurun_out/r2_pytest_gpu_full.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_fbb_tc|k_fbb_tma" -s 2 -c 2 -o gpurun_out/r2_ncu_fbb_products python bench.py --workload products --steps 1 --warmup 3 --no-cpu-baseline --no-clocks > /dev/null 2>&1
BG_FBB=tma timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_fbb_tma" -s 1 -c 1 -o gpurun_out/r2_ncu_fbb_products_tma python bench.py --workload products --steps 1 --warmup 3 --no-cpu-baseline --no-clocks > /dev/null 2>&1
ls gpurun_out/*.ncu-rep | tail -3
