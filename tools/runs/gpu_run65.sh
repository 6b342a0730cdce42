# slab boundary-phase K4 chunk: default (24) vs 28 / 32 / 40 (one wave of items at 32)
for v in - bc28 bc32 bc40 -; do
  if [ "$v" = "-" ]; then unset VG_LIB_VARIANT; else export VG_LIB_VARIANT=$v; fi
  timeout 300 python tools/slab_timing.py 2>&1 | python -c "
import sys,ast
for l in sys.stdin:
    p,d=l.split(' ',1); d=ast.literal_eval(d); print('$v', p, round(d['per_rank_gpu_ms'],4))"
done
