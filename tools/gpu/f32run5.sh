python -m pytest tests -m gpu -x -q -k "tf32 or f32 or F32 or split" > gpurun_out/f5_tests.log 2>&1; tail -3 gpurun_out/f5_tests.log
for ps in 1 0; do
  FMM_TF32_PRESPLIT=$ps timeout 600 python bench.py --dtype f32 --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/f5_bench_ps$ps.json 2> gpurun_out/f5_bench_ps$ps.err
  python -c "import json;d=json.load(open('gpurun_out/f5_bench_ps$ps.json'));print($ps, d['ms_per_step'],d['roofline']['launch_ms'],d['roofline']['step_share'],d['clocks']['sm_mhz'])"
done
