nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/fin_smi.txt
python -m pytest tests -m gpu -x -q > gpurun_out/fin_gputest.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/fin_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo "smoke rc $?"; cat gpurun_out/fin_smoke.log | tail -2
python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; echo "bench rc $?"
python -c "import json;d=json.load(open('gpurun_out/fin_bench.json'));print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['e2e']['value'],d['clocks'])"
python bench.py --impl reference > gpurun_out/fin_bench_ref.json 2> gpurun_out/fin_bench_ref.err; echo "ref rc $?"; cat gpurun_out/fin_bench_ref.json | head -c 600
