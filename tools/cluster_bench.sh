# Usage: bash tools/cluster_bench.sh "variant ..." — clustered stress bench line per build variant ("-" = in-tree lib)
for v in $1; do
  if [ "$v" = "-" ]; then unset VG_LIB_VARIANT; else export VG_LIB_VARIANT=$v; fi
  timeout 600 python bench.py --state clustered --steps 5 --warmup 3 --no-cpu-baseline --no-policy --no-e2e > gpurun_out/bclu_$v.json 2> gpurun_out/bclu_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/bclu_$v.json').read().strip().splitlines()[-1]); print('$v clustered', d['value'], d['ms_per_step'])"
done
