# LDF sort iteration: direct sort tests, sort timing per size, plan parity, config-2 plan microbench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sort.py -x -q > gpurun_out/sort_test.log 2>&1; tail -5 gpurun_out/sort_test.log
timeout 120 python tools/sort_bench.py 4096 8192 16384 32768
timeout 600 python -m pytest tests/test_gpu_plan_parity.py -x -q > gpurun_out/sort_parity.log 2>&1; tail -3 gpurun_out/sort_parity.log
timeout 300 python tools/plan_bench.py gpurun_out/plan_bench.json 2>&1 | tail -8
[ -f paper_2505_23022_b200/lib/libvar_lprof.so ] && SL_LIB_PATH=paper_2505_23022_b200/lib/libvar_lprof.so timeout 120 python tools/sort_prof.py 4096 32768 2>&1 | tail -4
