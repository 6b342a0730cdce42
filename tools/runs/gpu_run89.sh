# K4 uniform-register pair constants: single-world subset {slope, v/fov} in-tree; replica-instance subsets r6 / r5 / r3 vs all three (in-tree); GPU suite; bench c5
python paper_2207_03945_b200/_build.py --force > gpurun_out/build_89.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_89.log 2>&1; echo "tests rc $?"
grep -E "passed|failed" gpurun_out/gpu_tests_89.log | tail -3
VARS="r6 r5 r3 -" CFGS="c4" bash tools/ab.sh > gpurun_out/ab_89.txt 2>&1; cat gpurun_out/ab_89.txt
timeout 900 python bench.py > gpurun_out/bench_c5_89.json 2> gpurun_out/bench_c5_89.err; echo "bench c5 rc $?"
