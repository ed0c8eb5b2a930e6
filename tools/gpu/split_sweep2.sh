for c in C2 C4 C3; do
for sp in auto 0x070605 0x07060504 0x070603 0x070604 0x0706; do
  if [ $sp = auto ]; then unset FMM_K2F_SPLIT; else export FMM_K2F_SPLIT=$sp; fi
  python bench.py --config $c --steps 40 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c split $sp', round(d['ms_per_step'],4), round(d['roofline']['frac'],4))"
done; unset FMM_K2F_SPLIT; done
