# Round evidence in one gpurun call: GPU tests, smoke, default bench, reference arm,
# launch list of the default bench command, ncu --set full of the sweep kernel + plan kernels.
mkdir -p gpurun_out
nproc > gpurun_out/host_cores.txt; lscpu | grep "Model name" >> gpurun_out/host_cores.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> gpurun_out/host_cores.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -c 300 gpurun_out/bench_full.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 200 gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sl_sim_fast_kernel -c 1 -o gpurun_out/prof_full python bench.py --steps 1 --warmup 1 --no-cpu --no-plan > gpurun_out/prof_full.log 2>&1; tail -1 gpurun_out/prof_full.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"guard_admit|sort_warp|credit_select|plan_fused" -c 5 -o gpurun_out/prof_plan_scaled python tools/plan_only.py 65536 32 32 > gpurun_out/prof_plan_scaled.log 2>&1; tail -1 gpurun_out/prof_plan_scaled.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"guard_admit|sort_warp|credit_select|plan_fused" -c 8 -o gpurun_out/prof_plan_primary python tools/plan_only.py 1024 32 32 fused > gpurun_out/prof_plan_primary.log 2>&1; tail -1 gpurun_out/prof_plan_primary.log
ls gpurun_out
