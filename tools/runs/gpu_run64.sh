# K4 work-item cap for one large world 64 (in-tree) vs 128
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t64.log 2>&1; echo "tests rc $?"; tail -n1 gpurun_out/t64.log
VARS="- cm128" CFGS="c5 c4" timeout 1500 bash tools/ab.sh 2>&1
