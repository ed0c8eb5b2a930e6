# every C4 scaling mode with the fused-schedule tile sizing (FMM_SCALE_BIG=1, default) vs full-count tiles
python -m pytest tests/test_gpu_scaling.py -x -q -p no:cacheprovider > gpurun_out/big_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/big_tests.log
for s in outside inside out_in in_out repeated; do for b in 0 1; do
  FMM_SCALE_BIG=$b python bench.py --config C4 --scaling $s --steps 20 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());ss=d['roofline']['step_share'];print('$s big $b', round(d['ms_per_step'],4), 'SCALE', round(ss.get('SCALE',0),4), round(ss.get('SCALE',0)*d['ms_per_step']*1000,1),'us')"
done; done
