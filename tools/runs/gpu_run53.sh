# K4: the window-end test folded into the candidate predicate (NONAN) vs NaN positions (nn0)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t53.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/t53.log
VARS="- nn0" CFGS="c5 c4" timeout 2400 bash tools/ab.sh 2>&1
