# K4 8-byte ring entries (E8) for flock sector vision: full GPU suite, then A/B
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t37.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/t37.log
VARS="- e8off e8h2 e8h3" CFGS="c5 c4" timeout 2000 bash tools/ab.sh 2>&1
