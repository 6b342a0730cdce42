timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_r2d.log 2>&1; echo "tests rc $?"
tail -3 gpurun_out/gpu_tests_r2d.log
VARS="- atan5" CFGS="c5 c4 c3" timeout 1200 bash tools/ab.sh > gpurun_out/ab_r2d.txt 2>&1
cat gpurun_out/ab_r2d.txt
