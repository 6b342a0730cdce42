# k_sense overflow CTAs capped at one wave (looping over items) — full GPU suite, then A/B
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t35.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/t35.log
for v in - ow0 ow2; do
  if [ "$v" = "-" ]; then unset VG_LIB_VARIANT; else export VG_LIB_VARIANT=$v; fi
  timeout 300 python tools/slab_timing.py 2>&1 | sed "s/^/$v slab /"
done
unset VG_LIB_VARIANT
VARS="- ow0" CFGS="c5 c4 c2" timeout 1500 bash tools/ab.sh 2>&1
