# K4 HFORCE on c4: 2 (in-tree) vs 1 vs 3
VARS="- hf1 hf3" CFGS="c4" timeout 1500 bash tools/ab.sh 2>&1
