# K4 candidate loads at immediate offsets from one per-chunk pointer (xp) vs in-tree
python paper_2207_03945_b200/_build.py --force > gpurun_out/build_90.log 2>&1
VARS="xp -" CFGS="c5 c4" bash tools/ab.sh > gpurun_out/ab_90.txt 2>&1; cat gpurun_out/ab_90.txt
