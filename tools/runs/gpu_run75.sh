# K4: candidate loads of the first two halves unpredicated (in-tree) vs predicated (prev3)
VARS="- prev3" CFGS="c5 c4" timeout 1500 bash tools/ab.sh 2>&1
