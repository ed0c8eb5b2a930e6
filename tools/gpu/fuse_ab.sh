# fused A pass (FMM_SCALE_FUSE=1, default) vs the unfused passes: scaling tests, then C4 repeated A/B
python -m pytest tests/test_gpu_scaling.py -x -q -p no:cacheprovider > gpurun_out/fuse_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/fuse_tests.log
for f in 0 1 0 1; do
  FMM_SCALE_FUSE=$f python bench.py --config C4 --scaling repeated --steps 20 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());ss=d['roofline']['step_share'];print('fuse $f', round(d['ms_per_step'],4), 'SCALE', round(ss.get('SCALE',0),4), round(ss.get('SCALE',0)*d['ms_per_step']*1000,1),'us', d.get('scaling_steps'))"
done
for f in 0 1; do FMM_SCALE_FUSE=$f bash tools/gpu/scale_trace.sh; done
