# K4 on the uniform-register kernel: HFORCE 3 / 4 and 6 E8 halves vs in-tree (HFORCE 2, 4 halves)
python paper_2207_03945_b200/_build.py --force > gpurun_out/build_79.log 2>&1
VARS="hf3 hf4 e8h6 -" CFGS="c5 c4" bash tools/ab.sh > gpurun_out/ab_79.txt 2>&1; cat gpurun_out/ab_79.txt
