# round-2 final evidence: GPU tests, smoke, default bench (all legs), reference arm,
# --gpus 2 refusal, ncu of the hot sweep kernel (-> sim_kernel_ncu.json), launch list,
# ncu of the config-2 plan kernels (stress / primary), phase stamps of the stress guard
bash tools/gpu_r2b.sh > gpurun_out/r2b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sl_sim_fast_kernel -c 1 -o gpurun_out/prof_full python bench.py --steps 1 --warmup 0 --no-cpu --no-plan --no-config4 --no-report --no-baselines > gpurun_out/prof_full.log 2>&1
python tools/ncu_to_json.py gpurun_out/prof_full.ncu-rep 10000 4096 gpurun_out/sim_kernel_ncu.json
python tools/ncu_summary.py gpurun_out/prof_full.ncu-rep 222326173 > gpurun_out/prof_full.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/launches.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launches.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sort_cluster|guard_admit|credit_select" -o gpurun_out/prof_plan_stress python tools/plan_only.py 1 32768 32768 > gpurun_out/prof_plan_stress.log 2>&1
python tools/ncu_plan_table.py gpurun_out/prof_plan_stress.ncu-rep "stress 1x(32768+32768), r02 final (pipelined walk, certified folds)" > gpurun_out/plan_stress.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"guard_admit|sort_warp|credit_select|plan_fused" -c 8 -o gpurun_out/prof_plan_primary python tools/plan_only.py 1024 32 32 fused > gpurun_out/prof_plan_primary.log 2>&1
python tools/ncu_plan_table.py gpurun_out/prof_plan_primary.ncu-rep "primary 1024x(32+32), r02 final" > gpurun_out/plan_primary.txt
SL_LIB_PATH=paper_2505_23022_b200/lib/libvar_lprof.so python tools/large_prof.py > gpurun_out/lprof.txt 2>&1
ls gpurun_out
