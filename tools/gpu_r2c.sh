bash tools/gpu_r2b.sh > gpurun_out/r2b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sl_sim_fast_kernel -c 1 -o gpurun_out/prof_full python bench.py --steps 1 --warmup 0 --no-cpu --no-plan --no-config4 --no-report --no-baselines > gpurun_out/prof_full.log 2>&1; tail -1 gpurun_out/prof_full.log
python tools/ncu_to_json.py gpurun_out/prof_full.ncu-rep 10000 4096 gpurun_out/sim_kernel_ncu.json
python tools/ncu_summary.py gpurun_out/prof_full.ncu-rep 222326173 > gpurun_out/prof_full.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/launches.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launches.txt
