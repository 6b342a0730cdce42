# Usage: VARS="- variant" CFGS="c2 c3" bash tools/ab.sh   (variant "-" = in-tree lib; 3 alternating repeats)
for rep in 1 2 3; do for v in $VARS; do for c in $CFGS; do
  if [ "$v" = "-" ]; then unset VG_LIB_VARIANT; else export VG_LIB_VARIANT=$v; fi
  python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-policy 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
st=' '.join(f'{k.split()[0]}={v[\"ms\"]*1e3:.1f}' for k,v in d.get('stages',{}).items())
print('$v', '$c', $rep, round(d['ms_per_step']*1000,2), 'us |', st)"
done; done; done
