import torch, time
x = torch.rand(1080, 1920, 3).pin_memory()
y = torch.empty_like(x, device="cuda")
for _ in range(3): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): y.copy_(x, non_blocking=True)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"H2D 24.9MB: {ms:.3f} ms -> {x.numel()*4/ms/1e6:.1f} GB/s")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    e0.record(s)
    for _ in range(20): y.copy_(x, non_blocking=True)
    e1.record(s)
torch.cuda.synchronize(); print("side stream", e0.elapsed_time(e1)/20)
