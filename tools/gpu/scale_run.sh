python -m pytest tests/test_gpu_scaling.py -x -q > gpurun_out/sc_tests.log 2>&1; tail -2 gpurun_out/sc_tests.log
for v in "0 1" "1 2" "1 4" "1 8" "1 16"; do
  set -- $v
  FMM_SCALE_DYN=$1 FMM_SCALE_TPB=$2 python bench.py --config C4 --scaling repeated --steps 20 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());ss=d['roofline']['step_share'];print('dyn $1 tpb $2', round(d['ms_per_step'],4), 'SCALE', round(ss.get('SCALE',0),4), round(ss.get('SCALE',0)*d['ms_per_step']*1000,1),'us')"
done
