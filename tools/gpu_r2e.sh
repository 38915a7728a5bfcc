bash tools/gpu_r2b.sh > gpurun_out/r2b.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sort_cluster|guard_admit|credit_select" -o gpurun_out/prof_plan_stress python tools/plan_only.py 1 32768 32768 > gpurun_out/prof_plan_stress.log 2>&1
python tools/ncu_plan_table.py gpurun_out/prof_plan_stress.ncu-rep "stress 1x(32768+32768), r02 final (16-CTA select)" > gpurun_out/plan_stress.txt
