# One bench line per workload (README table): python bench.py for c1..c5, ray, clustered.
set -u
out=gpurun_out/bench_all.jsonl; : > $out
for c in c1 c2 c3 c4 c5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-policy 2>/dev/null | tail -1 >> $out
done
timeout 900 python bench.py --vision ray --no-cpu-baseline --no-policy 2>/dev/null | tail -1 >> $out
timeout 900 python bench.py --state clustered --steps 10 --no-cpu-baseline --no-policy 2>/dev/null | tail -1 >> $out
wc -l $out
