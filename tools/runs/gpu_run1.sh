set -x
nproc
python paper_2207_03945_b200/_build.py --force > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/gpu_tests_r2a.log 2>&1; echo "tests rc $?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c5_r2a.json 2> gpurun_out/bench_c5_r2a.err; echo "bench rc $?"
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-policy --no-cpu-baseline > gpurun_out/bench_c4_r2a.json 2> gpurun_out/bench_c4_r2a.err; echo "bench c4 rc $?"
tail -5 gpurun_out/gpu_tests_r2a.log
