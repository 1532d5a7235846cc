"""Burst vs sustained HBM copy bandwidth on this box (diagnostic for the roofline)."""
import torch, time
a = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
b = torch.empty_like(a)
a.normal_()
for _ in range(5):
    b.copy_(a)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); b.copy_(a); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
n = 1500
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n):
    b.copy_(a)
e1.record(); torch.cuda.synchronize()
sus = e0.elapsed_time(e1) / n
byt = 2 * a.numel() * 2
print(f"burst {byt / best / 1e6:.1f} GB/s  sustained({n} copies, {e0.elapsed_time(e1)/1e3:.1f} s) {byt / sus / 1e6:.1f} GB/s")
