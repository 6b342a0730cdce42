# Usage: bash tools/ray_ab.sh "variant ..." — ray-vision bench (2 runs) per build variant ("-" = in-tree lib)
for v in $1; do
  if [ "$v" = "-" ]; then unset VG_LIB_VARIANT; else export VG_LIB_VARIANT=$v; fi
  for i in 1 2; do
  python bench.py --vision ray --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-policy > gpurun_out/br_$v.json 2>gpurun_out/br_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/br_$v.json').read().strip().splitlines()[-1]); print('$v ray', d['value'], d['ms_per_step'])"
  done
done
