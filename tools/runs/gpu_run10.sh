B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-c4-binning"
$B --config c4 --no-policy > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_replica_bin -s 2 -c 1 -o gpurun_out/prof_rb_r2 -f $B --config c4 --no-policy > gpurun_out/ncu_rb.log 2>&1; echo "rb $?"
ncu --set full --clock-control none --import-source on -k regex:k_sense -s 3 -c 1 -o gpurun_out/prof_k4_r2 -f $B --no-policy > gpurun_out/ncu_k4.log 2>&1; echo "k4 $?"
ncu --set full --clock-control none --import-source on -k regex:k_policy -s 3 -c 1 -o gpurun_out/prof_k7_r2 -f $B > gpurun_out/ncu_k7.log 2>&1; echo "k7 $?"
ls -la gpurun_out/*.ncu-rep
