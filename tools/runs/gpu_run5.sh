timeout 900 python -m pytest tests/test_slab.py -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_slab_r2e.log 2>&1; echo "slab rc $?"
tail -15 gpurun_out/gpu_slab_r2e.log
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_r2e.log 2>&1; echo "tests rc $?"
tail -3 gpurun_out/gpu_tests_r2e.log
timeout 300 python tools/slab_timing.py > gpurun_out/slab_timing_r2e.txt 2>&1; tail -20 gpurun_out/slab_timing_r2e.txt
