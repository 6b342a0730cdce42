# K4 DEF = 2 instance for one large world (HFORCE_SINGLE 3, in-tree) vs 2 (hs2); GPU suite
python paper_2207_03945_b200/_build.py --force > gpurun_out/build_81.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_81.log 2>&1; echo "tests rc $?"
grep -E "passed|failed" gpurun_out/gpu_tests_81.log | tail -3
VARS="hs2 -" CFGS="c5 c4 c2 c3" bash tools/ab.sh > gpurun_out/ab_81.txt 2>&1; cat gpurun_out/ab_81.txt
