# final evidence at K4 v22 + aligned drain batches
# Round-2 evidence run (one B200): GPU tests, parity statistics, bench lines, slab timing,
# ncu launch lists and full captures.  Everything lands in gpurun_out/.
python paper_2207_03945_b200/_build.py --force > gpurun_out/build_r2.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_r2.log 2>&1; echo "tests rc $?"
grep -E "passed|failed" gpurun_out/gpu_tests_r2.log | tail -3
timeout 900 python bench.py > gpurun_out/bench_c5_r2.json 2> gpurun_out/bench_c5_r2.err; echo "bench c5 rc $?"
timeout 600 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4_r2.json 2> gpurun_out/bench_c4_r2.err; echo "bench c4 rc $?"
timeout 1200 python tools/parity_stats.py > gpurun_out/parity_stats_r2.log 2>&1; echo "parity rc $?"
cp profiles/parity_stats.json gpurun_out/parity_stats_r2.json
timeout 300 python tools/slab_timing.py > gpurun_out/slab_timing_r2.txt 2>&1; echo "slab rc $?"
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-policy --no-c4-binning"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5_r2.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "launches rc $?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c4_r2.csv $B --config c4 > gpurun_out/ncu_launch4.log 2>&1; echo "launches c4 rc $?"
ncu --set full --clock-control none --import-source on -k regex:k_sense -s 3 -c 1 -o gpurun_out/prof_k4_r2b -f $B > gpurun_out/ncu_k4.log 2>&1; echo "k4 $?"
ncu --set full --clock-control none --import-source on -k regex:k_replica_bin -s 2 -c 1 -o gpurun_out/prof_rb_r2b -f $B --config c4 > gpurun_out/ncu_rb.log 2>&1; echo "rb $?"
ncu --set full --clock-control none --import-source on -k regex:k_policy -s 3 -c 1 -o gpurun_out/prof_k7_r2b -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-c4-binning > gpurun_out/ncu_k7.log 2>&1; echo "k7 $?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_slab8_r2.csv python tools/slab8_launches.py 8 > gpurun_out/slab8_r2.log 2>&1; echo "slab8 launches rc $?"
