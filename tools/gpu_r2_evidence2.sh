# round-2 evidence (final code): launch list of the default bench, ncu --set full of the hot sweep
# kernel (-> sim_kernel_ncu.json), ncu of the config-2 plan kernels at the stress, scaled and primary shapes
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/launches.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launches.txt; head -30 gpurun_out/launches.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sl_sim_fast_kernel -c 1 -o gpurun_out/prof_full python bench.py --steps 1 --warmup 0 --no-cpu --no-plan --no-config4 --no-report --no-baselines > gpurun_out/prof_full.log 2>&1; tail -1 gpurun_out/prof_full.log
python tools/ncu_to_json.py gpurun_out/prof_full.ncu-rep 10000 4096 gpurun_out/sim_kernel_ncu.json; cat gpurun_out/sim_kernel_ncu.json
python tools/ncu_summary.py gpurun_out/prof_full.ncu-rep 222326173 > gpurun_out/prof_full.txt 2>&1; head -25 gpurun_out/prof_full.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sort_cluster|guard_admit|credit_select" -o gpurun_out/prof_plan_stress python tools/plan_only.py 1 32768 32768 > gpurun_out/prof_plan_stress.log 2>&1; tail -1 gpurun_out/prof_plan_stress.log
python tools/ncu_plan_table.py gpurun_out/prof_plan_stress.ncu-rep "stress 1x(32768+32768), r02 final" > gpurun_out/plan_stress.txt; cat gpurun_out/plan_stress.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"guard_admit|sort_warp|credit_select|plan_fused" -c 8 -o gpurun_out/prof_plan_scaled python tools/plan_only.py 262144 32 32 fused > gpurun_out/prof_plan_scaled.log 2>&1; tail -1 gpurun_out/prof_plan_scaled.log
python tools/ncu_plan_table.py gpurun_out/prof_plan_scaled.ncu-rep "scaled 262144x(32+32), r02 final" > gpurun_out/plan_scaled.txt; cat gpurun_out/plan_scaled.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"guard_admit|sort_warp|credit_select|plan_fused" -c 8 -o gpurun_out/prof_plan_primary python tools/plan_only.py 1024 32 32 fused > gpurun_out/prof_plan_primary.log 2>&1; tail -1 gpurun_out/prof_plan_primary.log
python tools/ncu_plan_table.py gpurun_out/prof_plan_primary.ncu-rep "primary 1024x(32+32), r02 final" > gpurun_out/plan_primary.txt; cat gpurun_out/plan_primary.txt
ls gpurun_out
