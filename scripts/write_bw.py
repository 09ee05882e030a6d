import torch
n = 10_510_000_000 // 8
x = torch.empty(n, dtype=torch.float64, device="cuda")
def t(f, reps=5):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
ms = t(lambda: x.fill_(1.5)); print(f"fill_ {ms:.3f} ms {n*8/ms/1e6:.0f} GB/s")
ms = t(lambda: x.zero_()); print(f"zero_ {ms:.3f} ms {n*8/ms/1e6:.0f} GB/s")
y = torch.empty_like(x)
ms = t(lambda: y.copy_(x)); print(f"copy_ {ms:.3f} ms {2*n*8/ms/1e6:.0f} GB/s (r+w)")
ms = t(lambda: x.sum()); print(f"sum {ms:.3f} ms {n*8/ms/1e6:.0f} GB/s")
