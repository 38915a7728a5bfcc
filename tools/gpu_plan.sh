# config-2 plan kernels: parity tests + microbench table
timeout 600 python -m pytest tests/test_gpu_plan_parity.py -x -q 2>&1 | tail -1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-config4 --no-report 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k,v in d['config2_plan_step'].items(): print(k, {kk:(round(vv['us'],1), round(vv['frac'],3)) for kk,vv in v['kernels'].items()})"
