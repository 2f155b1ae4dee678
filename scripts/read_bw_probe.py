"""Read bandwidth ceilings on this B200: torch reduction over the Reddit X
(561 MB fp32) and a copy, CUDA events, best of 10."""
import torch
x = torch.rand(232965, 602, device="cuda")
y = torch.empty_like(x)
def t(f):
    best = 1e9
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best
nb = x.numel() * 4
ts = t(lambda: x.sum())
tc = t(lambda: y.copy_(x))
print(f"sum: {ts*1e3:.1f} us, {nb/ts/1e6:.0f} GB/s read; copy: {tc*1e3:.1f} us, {2*nb/tc/1e6:.0f} GB/s r+w")
