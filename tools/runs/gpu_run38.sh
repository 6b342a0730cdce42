# K4 E8: halves per chunk 4 (in-tree) vs 5 / 6 / 7
VARS="- e8h5 e8h6 e8h7" CFGS="c5 c4" timeout 2000 bash tools/ab.sh 2>&1
