# slab P = 2/4/8 per-rank: K4 items per resident-CTA slot 4 (in-tree) / 2 / 1, with and without
# the batched window pass in slab ranks
for v in - ips2 ips1 ips2w ips1w -; do
  if [ "$v" = "-" ]; then unset VG_LIB_VARIANT; else export VG_LIB_VARIANT=$v; fi
  timeout 300 python tools/slab_timing.py 2>&1 | python -c "
import sys,ast
for l in sys.stdin:
    p,d=l.split(' ',1); d=ast.literal_eval(d); print('$v', p, round(d['per_rank_gpu_ms'],4))"
done
