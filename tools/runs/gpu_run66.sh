# K4 default-constant instance at 9 / 10 CTAs per SM (56 / 48 registers) vs 8 (64)
VARS="- mb9 mb10" CFGS="c5 c4" timeout 1500 bash tools/ab.sh 2>&1
