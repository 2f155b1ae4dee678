# one ncu --set full capture of each hot kernel (one launch each) on the Reddit-shape bench
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_KERNELS:-k_bmm_imma|k_sl_bb|k_sl_gcn1<}" -c ${NCU_COUNT:-3} \
  -o gpurun_out/${NCU_NAME:-full} -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-clocks > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
