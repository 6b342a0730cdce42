./tools/probes/tanh_probe > gpurun_out/tanh_probe.txt 2>&1; cat gpurun_out/tanh_probe.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_r2f.log 2>&1; echo "tests rc $?"
grep -E "passed|failed|FAILED|Error" gpurun_out/gpu_tests_r2f.log | tail -12
VARS="- rbs1 rbs2 rb512" CFGS="c4" timeout 900 bash tools/ab.sh > gpurun_out/ab_r2f.txt 2>&1
cat gpurun_out/ab_r2f.txt
