# K4 flock pair-pass constants in uniform registers (uc: VG_SENSE_UCONST=1) vs in-tree
python paper_2207_03945_b200/_build.py --force > gpurun_out/build_86.log 2>&1
VARS="uc -" CFGS="c5 c4" bash tools/ab.sh > gpurun_out/ab_86.txt 2>&1; cat gpurun_out/ab_86.txt
