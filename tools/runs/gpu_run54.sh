# K4: the self-slot test only in the run holding the queries' own cell (OWNRUN) vs every run
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t54.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/t54.log
VARS="- ow0" CFGS="c5 c4" timeout 2400 bash tools/ab.sh 2>&1
