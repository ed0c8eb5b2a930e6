for gm in 16 1 8 32; do
  FMM_TF32_GROUP_M=$gm timeout 600 python bench.py --dtype f32 --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/f3_bench_gm$gm.json 2> gpurun_out/f3_bench_gm$gm.err
  python -c "import json;d=json.load(open('gpurun_out/f3_bench_gm$gm.json'));print($gm, d['ms_per_step'],d['roofline']['launch_ms'],d['clocks']['sm_mhz'])"
done
for gm in 16 1; do
FMM_TF32_GROUP_M=$gm timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k2p -c 1 python tools/tf32_leaf_probe.py 8192 > gpurun_out/f3_ncu_gm$gm.log 2>&1 || tail -20 gpurun_out/f3_ncu_gm$gm.log
done
