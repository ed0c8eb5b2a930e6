set -x
python -m pytest tests -m gpu -x -q -k "node_st or recursion or parity" > gpurun_out/pt.log 2>&1; echo pytest=$?
for v in 1 2 3 4 5 6; do FMM_K1_VARIANT=$v python tools/bench_passes.py >> gpurun_out/passes.log 2>&1; done
for v in 1 2 3 5; do for c in C2 C4; do echo "v=$v $c" >> gpurun_out/cfg.log; FMM_K1_VARIANT=$v python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['step_share'])" >> gpurun_out/cfg.log 2>&1; done; done
