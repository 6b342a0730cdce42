# K4 at v22 + RINGB: single-world constant subsets all three (s7) / slope only (s2b) vs {slope, v/fov} (in-tree)
python paper_2207_03945_b200/_build.py --force > gpurun_out/build_95.log 2>&1
VARS="s7 s2b -" CFGS="c5" bash tools/ab.sh > gpurun_out/ab_95.txt 2>&1; cat gpurun_out/ab_95.txt
