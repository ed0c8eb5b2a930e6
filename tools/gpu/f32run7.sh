export FMM_TF32_PAIR=1
timeout 60 python tools/tf32_leaf_probe.py 1024 > gpurun_out/f7_probe.txt 2>&1; echo "probe rc $?"; cat gpurun_out/f7_probe.txt | tail -3
timeout 300 python -m pytest tests -m gpu -x -q -k "tf32 or f32 or F32 or split" > gpurun_out/f7_tests.log 2>&1; echo "tests rc $?"; tail -15 gpurun_out/f7_tests.log
timeout 120 python tools/tf32_leaf_probe.py 8192
timeout 600 python bench.py --dtype f32 --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/f7_bench.json 2> gpurun_out/f7_bench.err
python -c "import json;d=json.load(open('gpurun_out/f7_bench.json'));print(d['ms_per_step'],d['roofline']['launch_ms'],d['roofline']['step_share'],d['clocks']['sm_mhz'])"
