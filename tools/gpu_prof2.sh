bash tools/gpu_iter.sh
timeout 300 ncu --set full --import-source on -k regex:sl_sim_fast -c 1 -o gpurun_out/prof_single python bench.py --rates 1 --scales 1 --steps 1 --warmup 1 --no-cpu --no-plan > gpurun_out/prof_single.log 2>&1; tail -1 gpurun_out/prof_single.log
timeout 900 ncu --set full --import-source on -k regex:sl_sim_fast -c 1 -o gpurun_out/prof_full python bench.py --steps 1 --warmup 1 --no-cpu --no-plan > gpurun_out/prof_full.log 2>&1; tail -1 gpurun_out/prof_full.log
