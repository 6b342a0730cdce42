B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-c4-binning --no-policy"
ncu --set full --clock-control none --import-source on -k regex:k_replica_bin -s 2 -c 1 -o gpurun_out/prof_rb_r2c -f $B --config c4 > gpurun_out/ncu_rb.log 2>&1; echo "rb $?"
