# K4 runtime hforce (3 for one large world, 2 for replicas; in-tree) vs compile-time HFORCE 3 (hf3) vs 2 everywhere (hfs0); GPU suite
python paper_2207_03945_b200/_build.py --force > gpurun_out/build_80.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_80.log 2>&1; echo "tests rc $?"
grep -E "passed|failed" gpurun_out/gpu_tests_80.log | tail -3
VARS="hf3 hfs0 -" CFGS="c5 c4" bash tools/ab.sh > gpurun_out/ab_80.txt 2>&1; cat gpurun_out/ab_80.txt
