# K4 after the uniform-register change: HFORCE 1 (replicas), 2 / 3 E8 halves per chunk, single-world item cap 128 / 32, vs in-tree
python paper_2207_03945_b200/_build.py --force > gpurun_out/build_82.log 2>&1
VARS="hf1 e8h2 e8h3 cms128 cms32 -" CFGS="c5 c4" bash tools/ab.sh > gpurun_out/ab_82.txt 2>&1; cat gpurun_out/ab_82.txt
