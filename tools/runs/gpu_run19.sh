timeout 900 python -m pytest tests/test_slab.py -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_r2n.log 2>&1; echo "tests rc $?"
grep -E "passed|failed|FAILED|Error" gpurun_out/gpu_tests_r2n.log | tail -12
timeout 300 python tools/slab_timing.py > gpurun_out/slab_timing_r2n.txt 2>&1; tail -3 gpurun_out/slab_timing_r2n.txt
export VG_NO_GRAPH=1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_slab8b.csv python tools/slab8_launches.py 8 > gpurun_out/slab8.log 2>&1; echo "rc $?"
