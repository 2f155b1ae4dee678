# round evidence: GPU tests, smoke, full bench (with CPU baseline), launch list, ncu --set full of the hot kernels
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/ev_gpu.txt
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/ev_pytest.log
timeout 300 python __graft_entry__.py > gpurun_out/ev_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev_ref.json 2> gpurun_out/ev_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/ev_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-clocks > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fbb_tma|k_win_bb|k_bv_gcn1|k_sl_gcn1_records" -c 4 -o gpurun_out/ev_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-clocks > /dev/null 2>&1
cat gpurun_out/ev_pytest.log gpurun_out/ev_smoke.log | tail -4; python scripts/summ.py gpurun_out/ev_bench.json; head -c 600 gpurun_out/ev_ref.json
