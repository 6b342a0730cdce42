# K4 at v22 (pointer loads): replica HFORCE 3 (hf3), single-world HFORCE 4 (hs4), drain unroll 2 (du2) vs in-tree
python paper_2207_03945_b200/_build.py --force > gpurun_out/build_92.log 2>&1
VARS="hf3 hs4 du2 -" CFGS="c5 c4" bash tools/ab.sh > gpurun_out/ab_92.txt 2>&1; cat gpurun_out/ab_92.txt
