# measure pinned H2D / D2H bandwidth for the Reddit-shape X and output
import torch, time
torch.cuda.init()
x = torch.empty((232965, 602), dtype=torch.float32).pin_memory()
o = torch.empty((232965, 41), dtype=torch.float32).pin_memory()
dx = torch.empty_like(x, device="cuda"); do = torch.empty_like(o, device="cuda")
for name, src, dst in [("h2d X", x, dx), ("d2h out", do, o)]:
    for _ in range(3): dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10): dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) * 100
    print(name, round(ms, 3), "ms", round(src.numel() * 4 / ms / 1e6, 1), "GB/s")
