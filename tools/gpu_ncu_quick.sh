# quick ncu counters of the hot sweep kernel for each lib variant given as args
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active
for s in no_instruction wait short_scoreboard long_scoreboard lg_throttle math_pipe_throttle mio_throttle branch_resolving not_selected selected; do M=$M,smsp__average_warps_issue_stalled_${s}_per_issue_active.ratio; done
i=0
for v in "$@"; do
  i=$((i+1))
  SL_LIB_PATH=$v timeout 600 ncu --metrics $M -k regex:sl_sim_fast_kernel -c 1 --csv --log-file gpurun_out/nq_$i.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-plan > /dev/null 2>&1
  echo "== $v"
  python - gpurun_out/nq_$i.csv <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if r]
h = next(r for r in rows if "Metric Name" in r)
for r in rows[rows.index(h) + 1:]:
    d = dict(zip(h, r))
    print("   ", d["Metric Name"].replace("smsp__average_warps_issue_stalled_", "stall_"), d["Metric Value"], d["Metric Unit"])
PY
done
