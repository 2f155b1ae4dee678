cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_win_bb|k_bv_gcn1|k_fbb_tma" -s 5 -c 3 -o gpurun_out/r2_ncu1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-clocks > gpurun_out/r2_ncu1.log 2>&1
echo rc=$? >> gpurun_out/r2_ncu1.log
tail -3 gpurun_out/r2_ncu1.log
