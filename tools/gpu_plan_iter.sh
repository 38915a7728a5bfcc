mkdir -p gpurun_out
[ -f paper_2505_23022_b200/lib/libvar_lprof.so ] && SL_LIB_PATH=paper_2505_23022_b200/lib/libvar_lprof.so timeout 60 python tools/large_prof.py 2>&1 | tail -4
timeout 600 python -m pytest tests/test_gpu_plan_parity.py -x -q > gpurun_out/plan_parity.log 2>&1; tail -5 gpurun_out/plan_parity.log
timeout 300 python tools/plan_bench.py gpurun_out/plan_bench.json 2>&1 | tail -8
