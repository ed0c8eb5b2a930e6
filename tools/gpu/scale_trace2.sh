FMM_SCALE_TRACE=2 python - <<'PY' 2>&1 | grep scale | tail -14
import sys; sys.path.insert(0,'.')
import torch, bench, paper_1507_00687_b200 as fb
Ah,Bh = bench.make_inputs("C4","f64")
A,B = Ah.cuda(), Bh.cuda()
p = bench.make_plan(fb, "C4", scaling="repeated")
for _ in range(3): p.execute(A,B)
torch.cuda.synchronize()
PY
