for f in 0.0 0.005 0.01 0.02; do
  a=$(SL_LIB_PATH=paper_2505_23022_b200/lib/libvar_la.so SL_LOOKAHEAD_FRAC=$f timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --no-plan 2>/dev/null | python -c "import json,sys; print('%.1f' % json.loads(sys.stdin.readlines()[-1])['ms_per_step'])")
  echo "la lib lookahead_frac $f sweep_ms $a"
done
a=$(timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --no-plan 2>/dev/null | python -c "import json,sys; print('%.1f' % json.loads(sys.stdin.readlines()[-1])['ms_per_step'])")
echo "default sweep_ms $a"
