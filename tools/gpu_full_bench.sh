# Full round evidence: default bench, reference arm, launch list, ncu captures of the plan kernels.
nproc > gpurun_out/host_cores.txt; lscpu | grep "Model name" >> gpurun_out/host_cores.txt
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -c 600 gpurun_out/bench_full.json
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 300 gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --import-source on -k regex:"sort_warp|sort_tile|merge_pass|guard_admit|credit_select" -c 12 -o gpurun_out/prof_plan python bench.py --rates 2 --scales 2 --steps 1 --warmup 1 --no-cpu > gpurun_out/prof_plan.log 2>&1; tail -1 gpurun_out/prof_plan.log
