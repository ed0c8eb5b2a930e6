"""Read-bandwidth probe: torch reductions over a 4096 x 4096 FP64 matrix (the C4 operand size),
to calibrate the one-kernel scaling run's passes (one read of A and B per step)."""
import torch
x = torch.rand(4096, 4096, dtype=torch.float64, device="cuda")
y = torch.rand(4096, 4096, dtype=torch.float64, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
def t(fn, reps=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tot = 0.0
    for _ in range(reps):
        flush.fill_(1)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps
for name, fn in [("amax all (x)", lambda: x.abs().amax()),
                 ("sum (x)", lambda: x.sum()),
                 ("row max (x)", lambda: x.amax(dim=1)),
                 ("col max (x)", lambda: x.amax(dim=0)),
                 ("sum x + sum y", lambda: (x.sum(), y.sum())),
                 ("copy x->y", lambda: y.copy_(x))]:
    ms = t(fn)
    nb = 134217728 * (2 if ("y" in name and "copy" not in name) else 1) * (2 if "copy" in name else 1)
    print(f"{name:16s} {ms*1e3:8.1f} us  {nb/ms/1e6:7.0f} GB/s")
