# config-2 scaled plan kernels per lib variant (scan = guard_admit_group_kernel at >= 8192 segments)
for v in paper_2505_23022_b200/lib/libscorpio_b200.so paper_2505_23022_b200/lib/libvar_*.so; do
  SL_LIB_PATH=$v timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu --no-config4 --no-report 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['config2_plan_step']
print('$(basename $v)', {k: (round(v['kernels']['scan']['us'],1), round(v['kernels']['scan']['frac'],3)) for k,v in c.items() if k.startswith('scaled')})"
done
SL_LIB_PATH=$(ls paper_2505_23022_b200/lib/libvar_*.so | head -1) SL_PLAN_GROUP_MIN=1 timeout 600 python -m pytest tests/test_gpu_plan_parity.py -q 2>&1 | tail -1
