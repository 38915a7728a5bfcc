# sweep-kernel variants (lib/libvar_*.so given as args) vs the default build: config-3 sweep ms (3 runs each)
for v in paper_2505_23022_b200/lib/libscorpio_b200.so "$@"; do
  for r in 1 2; do
    b=$(SL_LIB_PATH=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-plan --no-config4 --no-report --no-baselines 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('%.2f' % d['roofline']['kernel_ms'])")
    echo "$(basename $v) sweep_kernel_ms $b"
  done
done
