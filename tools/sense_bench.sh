# Usage: bash tools/sense_bench.sh "variant1 variant2 ..." "c5 c4"   (variant "-" = in-tree lib)
VARS=${1:--}; CFGS=${2:-c5 c4}
for v in $VARS; do for c in $CFGS; do
  if [ "$v" = "-" ]; then unset VG_LIB_VARIANT; else export VG_LIB_VARIANT=$v; fi
  python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-policy > gpurun_out/sb_${v}_$c.json 2> gpurun_out/sb_${v}_$c.err || echo fail $v $c
done; done
unset VG_LIB_VARIANT
python - "$VARS" "$CFGS" <<'P'
import json, sys
for v in sys.argv[1].split():
    for c in sys.argv[2].split():
        try:
            d=json.loads(open(f"gpurun_out/sb_{v}_{c}.json").read().strip().splitlines()[-1])
            st=d.get("stages",{})
            print(f"{v:8s} {c} {d['value']:.3e} step {d['ms_per_step']:.4f} ms sense {st.get('sense',{}).get('ms')}")
        except Exception as e: print(v, c, "err", e)
P
