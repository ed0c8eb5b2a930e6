for ck in 128 256 512 128 256; do
  FMM_TF32_CHUNK=$ck python bench.py --dtype f32 --steps 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('chunk $ck', round(d['ms_per_step'],2), round(d['roofline']['launch_ms'],2), d['clocks']['sm_mhz'])"
done
for ck in 128 256 512; do FMM_TF32_CHUNK=$ck python tools/tf32_leaf_probe.py 4096; done
