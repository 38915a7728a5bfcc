# bench library variants (lib/libvar_*.so) against the default build: critical-path sim + sweep
for v in paper_2505_23022_b200/lib/libscorpio_b200.so paper_2505_23022_b200/lib/libvar_*.so; do
  a=$(SL_LIB_PATH=$v timeout 300 python bench.py --rates 1 --scales 1 --steps 2 --warmup 1 --no-cpu 2>/dev/null | python -c "import json,sys; print('%.1f' % json.loads(sys.stdin.readlines()[-1])['ms_per_step'])")
  b=$(SL_LIB_PATH=$v timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu 2>/dev/null | python -c "import json,sys; print('%.1f' % json.loads(sys.stdin.readlines()[-1])['ms_per_step'])")
  echo "$v single_ms $a sweep_ms $b"
done
