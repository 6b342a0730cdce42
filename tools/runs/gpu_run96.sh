# final smoke() + default bench at HEAD
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_96.log 2>&1; echo "smoke rc $?"; tail -3 gpurun_out/smoke_96.log
timeout 600 python bench.py > gpurun_out/bench_c5_96.json 2> gpurun_out/bench_c5_96.err; echo "bench rc $?"; tail -c 400 gpurun_out/bench_c5_96.json
