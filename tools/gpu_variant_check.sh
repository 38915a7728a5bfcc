# variant check: sweep parity tests under SL_LIB_PATH=$1, then sweep timing vs default, and the 2 req/s single-sim time
v=$1; shift
mkdir -p gpurun_out
SL_LIB_PATH=$v timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_sweep_parity.py tests/test_gpu_fullsize_parity.py -x -q > gpurun_out/variant_parity.log 2>&1; tail -2 gpurun_out/variant_parity.log
bash tools/gpu_variants_sweep.sh $v "$@"
for lib in paper_2505_23022_b200/lib/libscorpio_b200.so $v "$@"; do
  a=$(SL_LIB_PATH=$lib timeout 300 python bench.py --rates 1 --scales 1 --steps 3 --warmup 3 --no-cpu --no-plan --no-config4 --no-report --no-baselines 2>/dev/null | python -c "import json,sys; print('%.2f' % json.loads(sys.stdin.readlines()[-1])['roofline']['kernel_ms'])")
  echo "$(basename $lib) single_2rps_sim_ms $a"
done
