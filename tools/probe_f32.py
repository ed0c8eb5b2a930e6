"""C5 FP32 (3xTF32) plan timing probe with per-kind breakdown (device inputs)."""
import json, sys, time
sys.path.insert(0, '.')
import torch
import paper_1507_00687_b200 as fb
n = 32768
A = torch.rand(n, n, dtype=torch.float32, device="cuda") * 2 - 1
B = torch.rand(n, n, dtype=torch.float32, device="cuda") * 2 - 1
C = torch.empty_like(A)
w = fb.Rule.builtin("winograd")
p = fb.Plan([w, w, w], n, n, n, dtype="f32", leaf=fb.fmm.LEAF_3XTF32)
p.execute(A, B, C); torch.cuda.synchronize()
p.set_timing(True); p.step_times()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    p.execute(A, B, C)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
k = p.step_times()
print(json.dumps({"ms": round(ms, 2), "eff_tflops": round(2 * n ** 3 / ms / 1e9, 1),
                  "kinds_ms": {a: round(b[0] / 3, 2) for a, b in k.items()}}))
