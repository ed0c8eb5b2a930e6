# CUDA-graph replay vs direct launches for the small configs (bench --graph on / off)
for c in C1 C2 C4; do for g in on off on off; do
  python bench.py --config $c --graph $g --steps 50 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c graph $g', round(d['ms_per_step']*1000,2),'us')"
done; done
