# K4 work-item size cap 128 (in-tree: whole cells at c5) vs 64 / 40 queries
VARS="- cm64 cm40" CFGS="c5 c4" timeout 1500 bash tools/ab.sh 2>&1
