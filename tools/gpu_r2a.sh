# round-2 check: GPU tests, short bench (e2e through the API, cpu baselines), reference arm timing
mkdir -p gpurun_out
nproc > gpurun_out/host_cores.txt; lscpu | grep "Model name" >> gpurun_out/host_cores.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-plan --no-config4 --no-report --no-baselines > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err; tail -c 2500 gpurun_out/bench_a.json; tail -5 gpurun_out/bench_a.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_a.json 2> gpurun_out/bench_ref_a.err; cat gpurun_out/bench_ref_a.json; tail -5 gpurun_out/bench_ref_a.err
