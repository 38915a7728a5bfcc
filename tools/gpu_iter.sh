# Iteration check: critical-path sim alone, full sweep timing, then GPU parity tests (last line).
timeout 300 python bench.py --rates 1 --scales 1 --steps 3 --warmup 1 --no-cpu --no-plan 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('critical-path sim ms', round(d['ms_per_step'],2))"
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-plan > gpurun_out/bench_iter.json 2>gpurun_out/bench_iter.err; python -c "import json; d=json.load(open('gpurun_out/bench_iter.json')); print('sweep value %.3e ms %.1f frac %.3f' % (d['value'], d['ms_per_step'], d['roofline']['frac']))"
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
