python paper_2207_03945_b200/_build.py --force > gpurun_out/build_a.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_a.log 2>&1; echo "tests rc $?"
grep -E "passed|failed" gpurun_out/gpu_tests_a.log | tail -3
timeout 900 python bench.py > gpurun_out/bench_c5_a.json 2> gpurun_out/bench_c5_a.err; echo "bench c5 rc $?"
timeout 600 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4_a.json 2> gpurun_out/bench_c4_a.err; echo "bench c4 rc $?"
