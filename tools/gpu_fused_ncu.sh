# ncu --set full of the fused plan step at the config-2 primary shape (1024 x (32 + 32)) + sort tests
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sort.py -x -q > gpurun_out/sort_test.log 2>&1; tail -2 gpurun_out/sort_test.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:plan_fused -c 1 -o gpurun_out/fused python tools/plan_only.py 1024 32 32 fused > gpurun_out/fused_ncu.log 2>&1
ncu -i gpurun_out/fused.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warp_latency_per_inst_issued.ratio,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum > gpurun_out/fused_raw.csv 2>&1
cut -c1-700 gpurun_out/fused_raw.csv | tail -2
python tools/ncu_lines.py gpurun_out/fused.ncu-rep 45 > gpurun_out/fused_lines.txt 2>&1; head -55 gpurun_out/fused_lines.txt
