# ncu --set full of the cluster sort at W=4096 (1 CTA) and W=32768 (8-CTA cluster)
mkdir -p gpurun_out
for w in 4096 32768; do
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sort_cluster -c 1 -o gpurun_out/sort_$w python tools/sort_bench.py $w > gpurun_out/sort_ncu_$w.log 2>&1
ncu -i gpurun_out/sort_$w.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warp_latency_per_inst_issued.ratio,launch__registers_per_thread > gpurun_out/sort_raw_$w.csv 2>&1
cat gpurun_out/sort_raw_$w.csv | cut -c1-600 | tail -2
python tools/ncu_lines.py gpurun_out/sort_$w.ncu-rep 25 > gpurun_out/sort_lines_$w.txt 2>&1; head -40 gpurun_out/sort_lines_$w.txt
done
