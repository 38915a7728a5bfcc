for v in paper_2505_23022_b200/lib/libscorpio_b200.so paper_2505_23022_b200/lib/libvar_g*.so; do
  echo $v
  SL_LIB_PATH=$v timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu --no-config4 > gpurun_out/pf.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/pf.json'))
for k,v in d['config2_plan_step'].items(): print(' ', k, {kk: (round(vv['us'],1), round(vv['frac'],3)) for kk,vv in v['kernels'].items()})"
done
SL_PLAN_GROUP_MIN=1 timeout 600 python -m pytest tests/test_gpu_plan_parity.py -q 2>&1 | tail -1
