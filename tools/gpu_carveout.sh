# sweep time vs shared-memory carveout preference (SL_CARVEOUT percent; unset = driver default)
for r in 1 2; do
for c in default 0 10 20 25 50 100; do
  if [ $c = default ]; then unset SL_CARVEOUT; else export SL_CARVEOUT=$c; fi
  b=$(timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-plan --no-config4 --no-report 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('%.1f' % d['ms_per_step'])")
  echo "carveout $c sweep_ms $b"
done
done
