# every BASELINE config (C1-C4, C4 in all six scaling modes) through bench.py, one JSON line each
out=gpurun_out/cfg_bench_configs.jsonl
: > $out
for c in C1 C2 C2c C3; do
  timeout 600 python bench.py --config $c --steps 20 >> $out 2> gpurun_out/cfg_$c.err || echo "fail $c"
done
for s in none outside inside out_in in_out repeated; do
  timeout 600 python bench.py --config C4 --scaling $s --steps 20 >> $out 2> gpurun_out/cfg_C4_$s.err || echo "fail C4 $s"
done
python tools/bench_table.py $out
