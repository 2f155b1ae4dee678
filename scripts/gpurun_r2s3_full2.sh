cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s3b_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s3b_pytest_gpu.log
tail -3 gpurun_out/s3b_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/s3b_bench_reddit.json 2> gpurun_out/s3b_bench_reddit.err
for w in cora pubmed flickr products; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/s3b_bench_$w.json 2>gpurun_out/s3b_bench_$w.err; done
python -c "import __graft_entry__ as g; g.smoke()"
NCU_K="k_fbb_tmem" WL=reddit NAME=s3b_tmem2_reddit bash scripts/ncu_one.sh > /dev/null 2>&1
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_umma.py -x -q -k "tmem or bulk" > gpurun_out/s3b_memcheck.log 2>&1; tail -3 gpurun_out/s3b_memcheck.log
