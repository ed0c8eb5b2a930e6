# share of the blocks given to B's column tiles in the fused passes (FMM_SCALE_BFRAC)
for f in 0.5 0.45 0.4 0.5 0.45 0.4; do
  FMM_SCALE_BFRAC=$f python bench.py --config C4 --scaling repeated --steps 20 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());ss=d['roofline']['step_share'];print('bfrac $f', round(d['ms_per_step'],4), 'SCALE', round(ss.get('SCALE',0),4), round(ss.get('SCALE',0)*d['ms_per_step']*1000,1),'us')"
done
for f in 0.5 0.45 0.4; do echo "bfrac $f"; FMM_SCALE_BFRAC=$f timeout 100 bash tools/gpu/scale_trace2.sh | grep -E 'barriers|barrier  (2|6|10) '; done
