# K4: dynamic window batching, lane offsets by compare-count (in-tree) vs float (kitf)
VARS="- kitf" CFGS="c5 c4" timeout 2400 bash tools/ab.sh 2>&1
