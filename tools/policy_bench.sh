# Policy (K7) and rollout timing for the in-tree lib and tanh variants
# (tools/build_variants.py tanh1:-DVG_TANH_MODE=1 tanh2:-DVG_TANH_MODE=2)
for rep in 1 2; do for v in ${VARS:-- tanh1 tanh2}; do
  if [ "$v" = "-" ]; then unset VG_LIB_VARIANT; else export VG_LIB_VARIANT=$v; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pb_$v.json 2>gpurun_out/pb_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/pb_$v.json').read().strip().splitlines()[-1]); print('$v', $rep, d['policy']['ms'], d['policy']['hbm_frac'], d['rollout']['ms'])"
done; done
