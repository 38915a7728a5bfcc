# ncu source-level capture of the 16-segments-per-warp guard kernel at 262,144 segments
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:guard_admit_group -c 1 -o gpurun_out/group python tools/plan_only.py 262144 32 32 > gpurun_out/group.log 2>&1
ncu -i gpurun_out/group.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/group_src.csv 2>/dev/null
python tools/ncu_lines.py gpurun_out/group.ncu-rep 30 > gpurun_out/group_lines.txt 2>&1; head -40 gpurun_out/group_lines.txt
