# K4 single-world instance: subsets of the uniform-register pair constants (mask 1 atan c6, 2 tent slope, 4 v/fov) vs none (in-tree)
python paper_2207_03945_b200/_build.py --force > gpurun_out/build_88.log 2>&1
VARS="s1 s2 s4 s3 s6 s5 -" CFGS="c5" bash tools/ab.sh > gpurun_out/ab_88.txt 2>&1; cat gpurun_out/ab_88.txt
