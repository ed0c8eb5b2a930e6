set -x
python -m pytest tests -m gpu -x -q -k "tf32 or f32 or F32" > gpurun_out/f1_tests.log 2>&1; tail -3 gpurun_out/f1_tests.log
for cfg in 1 0 3 2; do FMM_TF32_CFG=$cfg timeout 120 python tools/tf32_leaf_probe.py 4096 >> gpurun_out/f1_probe.jsonl 2>>gpurun_out/f1_probe.err; done
for ck in 64 256 4096; do FMM_TF32_CHUNK=$ck timeout 120 python tools/tf32_leaf_probe.py 4096 >> gpurun_out/f1_probe.jsonl 2>>gpurun_out/f1_probe.err; done
cat gpurun_out/f1_probe.jsonl
timeout 600 python bench.py --dtype f32 --steps 5 --no-e2e > gpurun_out/f1_bench_f32.json 2> gpurun_out/f1_bench_f32.err
python -c "import json;d=json.load(open('gpurun_out/f1_bench_f32.json'));print(d['value'],d['ms_per_step'],d['roofline'],d['cpu_baseline'].get('error_vs_dd'),d['clocks'])"
