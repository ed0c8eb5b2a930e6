import torch
for n in (1 << 24, 1 << 26, 1 << 28):
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    for _ in range(3): x.sum()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): x.sum()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"sum of {n*8/1e6:8.0f} MB: {ms*1e3:8.1f} us  {n*8/ms/1e6:6.0f} GB/s")
    y = torch.empty_like(x)
    e0.record()
    for _ in range(10): y.copy_(x)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"copy of {n*8/1e6:8.0f} MB: {ms*1e3:8.1f} us  {2*n*8/ms/1e6:6.0f} GB/s (read+write)")
    del x, y
