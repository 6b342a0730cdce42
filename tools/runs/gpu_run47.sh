# K4: contact test, select and count under one predicate (PREDCNT) vs without
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t47.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/t47.log
VARS="- pc0" CFGS="c5 c4" timeout 2400 bash tools/ab.sh 2>&1
