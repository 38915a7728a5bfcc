for b in 1 2; do
  echo "blocks/SM=$b"; SL_BLOCKS_PER_SM=$b timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu --no-plan 2>/dev/null | python -c "import json,sys; print('sweep ms %.1f' % json.loads(sys.stdin.readlines()[-1])['ms_per_step'])"
  SL_BLOCKS_PER_SM=$b SL_LIB_PATH=paper_2505_23022_b200/lib/libvar_prof.so timeout 600 python tools/phase_prof.py 2>&1 | grep -A1 "longest"
done
