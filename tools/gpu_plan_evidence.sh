# ncu --set full of the config-2 plan kernels (final code): stress, scaled, primary shapes
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sort_cluster|guard_admit|credit_select" -o gpurun_out/prof_plan_stress python tools/plan_only.py 1 32768 32768 > gpurun_out/prof_plan_stress.log 2>&1; tail -1 gpurun_out/prof_plan_stress.log
python tools/ncu_plan_table.py gpurun_out/prof_plan_stress.ncu-rep "stress 1x(32768+32768), r02 final" > gpurun_out/plan_stress.txt; cat gpurun_out/plan_stress.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"guard_admit|sort_warp|credit_select|plan_fused" -c 8 -o gpurun_out/prof_plan_scaled python tools/plan_only.py 262144 32 32 fused > gpurun_out/prof_plan_scaled.log 2>&1; tail -1 gpurun_out/prof_plan_scaled.log
python tools/ncu_plan_table.py gpurun_out/prof_plan_scaled.ncu-rep "scaled 262144x(32+32), r02 final" > gpurun_out/plan_scaled.txt; cat gpurun_out/plan_scaled.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"guard_admit|sort_warp|credit_select|plan_fused" -c 8 -o gpurun_out/prof_plan_primary python tools/plan_only.py 1024 32 32 fused > gpurun_out/prof_plan_primary.log 2>&1; tail -1 gpurun_out/prof_plan_primary.log
python tools/ncu_plan_table.py gpurun_out/prof_plan_primary.ncu-rep "primary 1024x(32+32), r02 final" > gpurun_out/plan_primary.txt; cat gpurun_out/plan_primary.txt
