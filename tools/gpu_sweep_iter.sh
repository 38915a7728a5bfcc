# sweep-kernel iteration: parity tests of the simulation kernels + the config-3 bench line (no extras)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_sweep_parity.py tests/test_gpu_fullsize_parity.py -x -q > gpurun_out/sweep_parity.log 2>&1; tail -3 gpurun_out/sweep_parity.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-plan --no-config4 --no-report --no-baselines --no-cpu > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_sweep.json').read().strip().splitlines()[-1])
print('value %.3fG  ms %.2f  kernel_ms %.2f  e2e %.3fG' % (d['value']/1e9, d['ms_per_step'], d['roofline']['kernel_ms'], d['e2e']['value']/1e9))" || tail -5 gpurun_out/bench_sweep.err
