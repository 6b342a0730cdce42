# K4: loads of candidate halves wholly past the window end predicated off (LDPRED), with
# E8 four halves (static second sync) and with 16-byte entries
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t41.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/t41.log
VARS="- ldp e8off e8offldp" CFGS="c5 c4" timeout 2400 bash tools/ab.sh 2>&1
