# K4 ring drain loop unrolled by 2 (du2) vs in-tree
python paper_2207_03945_b200/_build.py --force > gpurun_out/build_84.log 2>&1
VARS="du2 -" CFGS="c5 c4" bash tools/ab.sh > gpurun_out/ab_84.txt 2>&1; cat gpurun_out/ab_84.txt
