# K4: the candidate test + push of both queries in one PTX block, window predicate shared (SCANASM)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t67.log 2>&1; echo "tests rc $?"; tail -n1 gpurun_out/t67.log
VARS="- sa0" CFGS="c5 c4" timeout 1500 bash tools/ab.sh 2>&1
