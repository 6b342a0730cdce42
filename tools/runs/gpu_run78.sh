# binning kernels with uniform-register warp/cell/count values (VG_BIN_UNI=1, in-tree) vs without (nobin): GPU suite + A/B c5/c4
python paper_2207_03945_b200/_build.py --force > gpurun_out/build_78.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_78.log 2>&1; echo "tests rc $?"
grep -E "passed|failed" gpurun_out/gpu_tests_78.log | tail -3
VARS="nobin -" CFGS="c5 c4" bash tools/ab.sh > gpurun_out/ab_78.txt 2>&1; cat gpurun_out/ab_78.txt
