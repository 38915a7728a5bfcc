timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python bench.py --rates 1 --scales 1 --steps 2 --warmup 1 --no-cpu 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('single-sim ms', d['ms_per_step'])"
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench4.json 2>gpurun_out/bench4.err; python -c "import json; d=json.load(open('gpurun_out/bench4.json')); print('value %.3e ms %.1f frac %.3f'%(d['value'],d['ms_per_step'],d['roofline']['frac']))"
