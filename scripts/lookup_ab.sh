# products forward with the 16-byte-store FBF lookup vs the scalar one; write ceiling of fill_
cd $GRAFT_REPO_ROOT
python - <<'P'
import torch
x = torch.empty(115_100_000, device="cuda")
for _ in range(3): x.fill_(1.0)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20): x.fill_(1.0)
b.record(); b.synchronize()
ms = a.elapsed_time(b) / 20
print("fill 460 MB: %.1f us  %.0f GB/s" % (ms * 1e3, x.numel() * 4 / ms / 1e6))
P
python -m pytest tests/test_gpu_layers.py tests/test_gpu_glue_layers.py tests/test_gpu_pair.py -x -q -m gpu 2>&1 | tail -1
for rep in 1 2 3; do
  for v in 0 1; do
    if [ $v = 1 ]; then export BG_LOOKUP_SCALAR=1; else unset BG_LOOKUP_SCALAR; fi
    echo "scalar=$v $(python bench.py --workload products --steps 20 --warmup 5 --no-cpu-baseline --no-clocks 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"])')"
  done
done
