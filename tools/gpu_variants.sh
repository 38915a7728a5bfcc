# bench the fast-kernel occupancy variants (lib/libscorpio_minb*.so)
for v in paper_2505_23022_b200/lib/libscorpio_b200.so paper_2505_23022_b200/lib/libscorpio_minb*.so; do
  SL_LIB_PATH=$v timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', 'ms %.1f'%d['ms_per_step'], 'value %.3e'%d['value'])"
done
SL_LIB_PATH=paper_2505_23022_b200/lib/libscorpio_minb4.so timeout 300 python bench.py --rates 1 --scales 1 --steps 2 --warmup 1 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('minb4 single-sim ms', d['ms_per_step'])"
