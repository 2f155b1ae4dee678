cd $GRAFT_REPO_ROOT
WL=products bash scripts/quick_bench.sh
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_fbb|k_bv_bb|k_bmm" -s 3 -c 4 -o gpurun_out/r2_ncu_products python bench.py --workload products --steps 1 --warmup 3 --no-cpu-baseline --no-clocks > gpurun_out/r2_ncu2.log 2>&1
echo rc=$? >> gpurun_out/r2_ncu2.log
tail -2 gpurun_out/r2_ncu2.log
