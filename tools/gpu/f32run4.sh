python -m pytest tests -m gpu -x -q -k "tf32 or f32 or F32" > gpurun_out/f4_tests.log 2>&1; tail -3 gpurun_out/f4_tests.log
for bmn in 1 0; do FMM_TF32_BMN=$bmn timeout 120 python tools/tf32_leaf_probe.py 8192; done
for bmn in 1 0; do
  FMM_TF32_BMN=$bmn timeout 600 python bench.py --dtype f32 --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/f4_bench_bmn$bmn.json 2> gpurun_out/f4_bench_bmn$bmn.err
  python -c "import json;d=json.load(open('gpurun_out/f4_bench_bmn$bmn.json'));print($bmn, d['ms_per_step'],d['roofline']['launch_ms'],d['clocks']['sm_mhz'])"
done
