# c5 binning: K1 counts without a returning atomic, K3 takes the slots from per-cell cursors
# (VG_BIN_RED) vs K1 returning the slots (red0)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t61.log 2>&1; echo "tests rc $?"; tail -n1 gpurun_out/t61.log
VARS="- red0" CFGS="c5" timeout 1500 bash tools/ab.sh 2>&1
