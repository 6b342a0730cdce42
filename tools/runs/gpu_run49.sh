# K4: runs without image shifts take their own chunk-loop instance (UNSH) vs not (un0)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t49.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/t49.log
VARS="- un0" CFGS="c5 c4" timeout 2400 bash tools/ab.sh 2>&1
