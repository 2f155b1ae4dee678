cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,pcie.link.gen.current,pcie.link.width.current --format=csv > gpurun_out/s3e_smi.txt
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s3e_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s3e_pytest_gpu.log
tail -3 gpurun_out/s3e_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/s3e_bench_reddit.json 2> gpurun_out/s3e_bench_reddit.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/s3e_ref_reddit.json 2> gpurun_out/s3e_ref_reddit.err
for w in cora pubmed flickr products; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/s3e_bench_$w.json 2>gpurun_out/s3e_bench_$w.err; done
python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s3e_launches_reddit.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-clocks > /dev/null 2>&1
echo done
NCU_K="k_fbf_lookup" NCU_SKIP=3 WL=products NAME=s3e_lookup_products bash scripts/ncu_one.sh > /dev/null 2>&1; echo ncu done
