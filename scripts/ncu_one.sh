# one ncu --set full capture: NCU_K (kernel regex), WL (workload), NAME; then the summary
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCU_K" -s ${NCU_SKIP:-2} -c ${NCU_COUNT:-1} \
  -o gpurun_out/$NAME -f python bench.py --workload ${WL:-reddit} --steps 1 --warmup 3 --no-cpu-baseline --no-clocks > gpurun_out/$NAME.log 2>&1
tail -2 gpurun_out/$NAME.log
python scripts/ncu_summary.py gpurun_out/$NAME.ncu-rep > gpurun_out/${NAME}_summary.txt 2>&1
cat gpurun_out/${NAME}_summary.txt
