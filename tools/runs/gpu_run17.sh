export VG_BENCH_GLOO_TEST=1
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533"
timeout 600 $T bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/gloo2_halo.json 2> gpurun_out/gloo2_halo.err; echo "halo rc $?"
timeout 600 $T bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --slab-scheme allgather > gpurun_out/gloo2_ag.json 2> gpurun_out/gloo2_ag.err; echo "ag rc $?"
timeout 600 $T bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --config c4 > gpurun_out/gloo2_c4.json 2> gpurun_out/gloo2_c4.err; echo "c4 rc $?"
for f in halo ag c4; do tail -c 600 gpurun_out/gloo2_$f.json; echo; tail -3 gpurun_out/gloo2_$f.err; done
