# K4: invisible flock pairs update a spare sector slot (no selects) vs the previous build
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t46.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/t46.log
VARS="- prev" CFGS="c5 c4" timeout 2400 bash tools/ab.sh 2>&1
