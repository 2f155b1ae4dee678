# quick GPU iteration: selected tests + bench (args: pytest selector)
mkdir -p gpurun_out
timeout 600 python -m pytest ${TESTS:-tests/test_gpu_window.py} -x -q 2>&1 | tail -15 > gpurun_out/pytest_quick.log
cat gpurun_out/pytest_quick.log
timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
tail -3 gpurun_out/bench_quick.err; cat gpurun_out/bench_quick.json
