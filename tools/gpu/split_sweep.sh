for c in C2 C4; do
for sp in auto 0 0x0704 0x0703 0x0705 0x070402 0x070503 0x0706 0x0702; do
  if [ $sp = auto ]; then unset FMM_K2F_SPLIT; else export FMM_K2F_SPLIT=$sp; fi
  python bench.py --config $c --steps 50 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c split $sp', round(d['ms_per_step'],4), round(d['roofline']['frac'],4))"
done; unset FMM_K2F_SPLIT; done
