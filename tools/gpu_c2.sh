timeout 600 python bench.py --no-cpu > gpurun_out/bench_full.json 2>gpurun_out/bench_full.err; tail -3 gpurun_out/bench_full.err
python -c "
import json; d=json.load(open('gpurun_out/bench_full.json')); print('sweep ms', round(d['ms_per_step'],1), d['value'], d['roofline']['frac'])
for k,v in d['config2_plan_step'].items(): print(k, round(v['us_per_step'],1), {kk: (round(vv['us'],1), round(vv['frac'],3)) for kk,vv in v['kernels'].items()})"
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
