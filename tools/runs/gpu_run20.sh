for v in - bc16 bc48 bc96; do
  if [ "$v" = "-" ]; then unset VG_LIB_VARIANT; else export VG_LIB_VARIANT=$v; fi
  echo "== $v"; timeout 300 python tools/slab_timing.py 2>&1 | tail -3
done
