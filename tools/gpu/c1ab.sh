cp paper_1507_00687_b200/csrc/kernels_small.cu tools/gpu/kernels_small_new.cu
run() { python bench.py --config C1 --steps $1 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$2 steps $1', round(d['ms_per_step']*1000,2),'us')"; }
run 200 new; run 20 new; run 200 new
cp tools/gpu/kernels_small_old.cu paper_1507_00687_b200/csrc/kernels_small.cu
python -m paper_1507_00687_b200.build > /dev/null 2>&1 || echo build-fail
run 200 old; run 20 old; run 200 old
cp tools/gpu/kernels_small_new.cu paper_1507_00687_b200/csrc/kernels_small.cu
