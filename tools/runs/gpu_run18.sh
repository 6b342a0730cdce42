export VG_NO_GRAPH=1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_slab8.csv python tools/slab8_launches.py 8 > gpurun_out/slab8.log 2>&1; echo "rc $?"
