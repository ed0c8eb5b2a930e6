python -m pytest tests/test_gpu_small.py tests/test_gpu_parity.py -x -q > gpurun_out/c1_tests.log 2>&1; tail -2 gpurun_out/c1_tests.log
for i in 1 2; do python bench.py --config C1 --steps 200 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['ms_per_step']*1e3,'us', d['roofline']['frac'])"; done
FMM_SMALL_TRACE=1 python tools/run_plan_once.py C1 --reps 5 2>&1 | tail -3
