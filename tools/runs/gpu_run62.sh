# K1: agents per thread 4 (in-tree) vs 1 / 2 / 8
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t62.log 2>&1; echo "tests rc $?"; tail -n1 gpurun_out/t62.log
VARS="- apt1 apt2 apt8" CFGS="c5 c3" timeout 1500 bash tools/ab.sh 2>&1
