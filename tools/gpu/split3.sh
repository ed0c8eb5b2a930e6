for c in C3 C3; do python bench.py --config $c --steps 40 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c auto', round(d['ms_per_step'],4))"; done
for sp in auto 0x0706 auto 0x0706; do
  if [ $sp = auto ]; then unset FMM_K2F_SPLIT; else export FMM_K2F_SPLIT=$sp; fi
  python bench.py --steps 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('C5 split $sp', round(d['ms_per_step'],2))"
done
