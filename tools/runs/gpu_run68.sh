# staged bin: the sense order placed in pass 2 from (cell, sub-bin) cursors (XO2) vs pass 3
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t68.log 2>&1; echo "tests rc $?"; tail -n1 gpurun_out/t68.log
VARS="- xo0" CFGS="c4" timeout 1500 bash tools/ab.sh 2>&1
