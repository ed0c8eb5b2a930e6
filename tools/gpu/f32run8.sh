for pr in 0 1 0 1; do
  FMM_TF32_PAIR=$pr timeout 600 python bench.py --dtype f32 --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/f8_bench_$pr.json 2> gpurun_out/f8_bench_$pr.err
  python -c "import json;d=json.load(open('gpurun_out/f8_bench_$pr.json'));print($pr, d['ms_per_step'],d['roofline']['launch_ms'],d['clocks']['sm_mhz'])"
done
nvidia-smi --query-gpu=power.limit,power.max_limit,temperature.gpu --format=csv
