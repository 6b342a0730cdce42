# K4: symmetric tent f = c_near - k |d - d_peak| (default constants: k_rise == k_fall) vs min(rise, fall)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t70.log 2>&1; echo "tests rc $?"; tail -n1 gpurun_out/t70.log
VARS="- ts0" CFGS="c5 c4" timeout 1500 bash tools/ab.sh 2>&1
timeout 900 python tools/parity_stats.py > gpurun_out/ps70.log 2>&1; echo "parity rc $?"; tail -5 gpurun_out/ps70.log
