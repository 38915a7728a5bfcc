# sweep-kernel variants vs default, 5 alternating runs each (kernel ms), for small differences
for r in 1 2 3 4 5; do
  for v in paper_2505_23022_b200/lib/libscorpio_b200.so "$@"; do
    b=$(SL_LIB_PATH=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-plan --no-config4 --no-report --no-baselines 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('%.2f' % d['roofline']['kernel_ms'])")
    echo "$(basename $v) $b"
  done
done
