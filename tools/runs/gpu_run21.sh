python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build21.log 2>&1; echo "build rc $?"
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2.log 2>&1; echo "smoke rc $?"; tail -3 gpurun_out/smoke_r2.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_r2o.log 2>&1; echo "tests rc $?"
grep -E "passed|failed|FAILED|Error" gpurun_out/gpu_tests_r2o.log | tail -5
