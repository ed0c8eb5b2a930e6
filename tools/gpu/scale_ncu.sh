# ncu --set full of the one-kernel scaling run at C4 (repeated), source-level stalls
cat > /tmp/sc1.py <<'PY'
import sys; sys.path.insert(0,'.')
import torch, bench, paper_1507_00687_b200 as fb
Ah,Bh = bench.make_inputs("C4","f64")
A,B = Ah.cuda(), Bh.cuda()
p = bench.make_plan(fb, "C4", scaling="repeated")
for _ in range(2): p.execute(A,B)
torch.cuda.synchronize()
PY
python /tmp/sc1.py && ncu --set full --import-source on --clock-control none -k regex:k_scale_coop -s 1 -c 1 -f -o gpurun_out/scale_final python /tmp/sc1.py > gpurun_out/scale_ncu.log 2>&1; echo ncu rc=$?; tail -3 gpurun_out/scale_ncu.log
