# K4: run windows of wn = 32 / nseg iterations per pass (in-tree) vs 5
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t58.log 2>&1; echo "tests rc $?"; tail -n1 gpurun_out/t58.log
VARS="- w5" CFGS="c5 c4" timeout 2400 bash tools/ab.sh 2>&1
