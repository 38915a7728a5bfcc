# Round evidence in one gpurun call: GPU tests, smoke, default bench, reference arm,
# launch list of the default bench command, ncu --set full of the sweep kernel + plan kernels.
set -x
mkdir -p gpurun_out
nproc > gpurun_out/host_cores.txt; lscpu | grep "Model name" >> gpurun_out/host_cores.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> gpurun_out/host_cores.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -c 1500 gpurun_out/bench_full.json
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 400 gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sl_sim_fast -c 1 -o gpurun_out/prof_full python bench.py --steps 1 --warmup 1 --no-cpu --no-plan > gpurun_out/prof_full.log 2>&1; tail -1 gpurun_out/prof_full.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sort_warp|sort_tile|merge_pass|guard_admit|credit_select" -c 12 -o gpurun_out/prof_plan python bench.py --rates 2 --scales 2 --steps 1 --warmup 1 --no-cpu > gpurun_out/prof_plan.log 2>&1; tail -1 gpurun_out/prof_plan.log
ls -la gpurun_out
