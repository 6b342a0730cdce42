# K4 default-constant instances at 7 CTAs per SM (72 registers, mb7) vs 8 (64, in-tree) on the uniform-register kernel
python paper_2207_03945_b200/_build.py --force > gpurun_out/build_85.log 2>&1
VARS="mb7 -" CFGS="c5 c4" bash tools/ab.sh > gpurun_out/ab_85.txt 2>&1; cat gpurun_out/ab_85.txt
