for f in 0.0 0.01 0.02 0.05; do
  a=$(SL_LOOKAHEAD_FRAC=$f timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --no-plan 2>/dev/null | python -c "import json,sys; print('%.1f' % json.loads(sys.stdin.readlines()[-1])['ms_per_step'])")
  echo "lookahead_frac $f sweep_ms $a"
done
timeout 300 python bench.py --rates 1 --scales 1 --steps 2 --warmup 1 --no-cpu --no-plan 2>/dev/null | python -c "import json,sys; print('single (flagged) ms %.1f' % json.loads(sys.stdin.readlines()[-1])['ms_per_step'])"
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
