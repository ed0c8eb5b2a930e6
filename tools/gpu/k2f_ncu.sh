for c in C2 C3; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k2f_gemm -c 1 -o gpurun_out/k2f_$c python tools/run_plan_once.py $c > gpurun_out/k2f_ncu_$c.log 2>&1 || tail -5 gpurun_out/k2f_ncu_$c.log
done
