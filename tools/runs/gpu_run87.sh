# K4 uniform-register pair-pass constants for the replica instance only (in-tree) vs none (uc0); GPU suite
python paper_2207_03945_b200/_build.py --force > gpurun_out/build_87.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_87.log 2>&1; echo "tests rc $?"
grep -E "passed|failed" gpurun_out/gpu_tests_87.log | tail -3
VARS="uc0 -" CFGS="c5 c4" bash tools/ab.sh > gpurun_out/ab_87.txt 2>&1; cat gpurun_out/ab_87.txt
timeout 600 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4_87.json 2> gpurun_out/bench_c4_87.err; echo "bench c4 rc $?"
timeout 900 python bench.py > gpurun_out/bench_c5_87.json 2> gpurun_out/bench_c5_87.err; echo "bench c5 rc $?"
