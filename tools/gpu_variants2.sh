# sweep time of lib variants (lib/libvar_*.so) vs the default build, interleaved, R rounds
R=${R:-3}
for r in $(seq $R); do
  for v in paper_2505_23022_b200/lib/libscorpio_b200.so paper_2505_23022_b200/lib/libvar_*.so; do
    b=$(SL_LIB_PATH=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-plan --no-config4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('%.1f %s' % (d['ms_per_step'], d['clocks']['sm_mhz']))")
    echo "$r $(basename $v) $b"
  done
done | sort -k2,2 -k1,1n | awk '{print} {m[$2]=(m[$2]==""||$3<m[$2])?$3:m[$2]} END {for (k in m) print "min", k, m[k]}'
