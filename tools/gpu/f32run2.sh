for cfg in 0 3 1; do
  FMM_TF32_CFG=$cfg timeout 600 python bench.py --dtype f32 --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/f2_bench_cfg$cfg.json 2> gpurun_out/f2_bench_cfg$cfg.err
  python -c "import json;d=json.load(open('gpurun_out/f2_bench_cfg$cfg.json'));print($cfg, d['ms_per_step'],d['roofline']['launch_ms'],d['clocks'])"
done
for cfg in 0 3; do
  FMM_TF32_CFG=$cfg timeout 300 ncu --set full --clock-control none -k regex:k2p -c 1 -o gpurun_out/f2_k2p_cfg$cfg python tools/tf32_leaf_probe.py 8192 > gpurun_out/f2_ncu_cfg$cfg.log 2>&1
done
