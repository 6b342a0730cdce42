# K4 on the final kernel: three halves per chunk (no second ring sync) / 8 warps per CTA
VARS="- e8h3 w8" CFGS="c5 c4" timeout 1500 bash tools/ab.sh 2>&1
