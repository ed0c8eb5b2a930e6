# L2 eviction-priority hints on the fused schedule's bulk copies (FMM_SCALE_L2HINT=1 default) vs none
python -m pytest tests/test_gpu_scaling.py -x -q -p no:cacheprovider > gpurun_out/hint_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/hint_tests.log
for h in 1 2 1 2; do
  FMM_SCALE_L2HINT=$h python bench.py --config C4 --scaling repeated --steps 20 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());ss=d['roofline']['step_share'];print('hint $h', round(d['ms_per_step'],4), 'SCALE', round(ss.get('SCALE',0),4), round(ss.get('SCALE',0)*d['ms_per_step']*1000,1),'us')"
done
for h in 1 2; do echo "hint $h"; FMM_SCALE_L2HINT=$h bash tools/gpu/scale_trace.sh; done
