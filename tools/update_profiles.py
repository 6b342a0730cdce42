"""Refresh the committed K4 evidence from a gpurun round:
    python tools/update_profiles.py TAG BENCH_JSON LAUNCHES_CSV NCU_REP "what changed"
Writes profiles/r1_bench_c5_TAG.json, profiles/r1_launches_c5_TAG.csv,
profiles/sense_traffic.json (DRAM bytes + warp instructions of k_sense, read by bench.py)
and appends a section to profiles/r1_ncu_summary.md."""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, bench, launches, rep, note = sys.argv[1:6]
P = os.path.join(ROOT, "profiles")
shutil.copy(bench, os.path.join(P, f"r1_bench_c5_{tag}.json"))
shutil.copy(launches, os.path.join(P, f"r1_launches_c5_{tag}.csv"))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout.splitlines()
rows = list(csv.reader(raw))
h = rows[0]
d = next(dict(zip(h, r)) for r in rows[2:] if "k_sense" in dict(zip(h, r))["Kernel Name"])
num = lambda k: float(d[k].replace(",", ""))
rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
unit = 1e6 if "Mbyte" in rows[1][h.index("dram__bytes_read.sum")] else 1.0
inst = num("smsp__inst_executed.sum")
pipes = {k.split("__")[1].split(".")[0]: num(k) for k in (
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active") if k in d}
json.dump({"config": "c5", "kernel": f"void k_sense<0, 1, 0, 0> ({tag})",
           "bytes_per_launch": (rd + wr) * unit, "dram_read_bytes": rd * unit,
           "dram_write_bytes": wr * unit, "warp_instructions": inst, "pct_of_peak": pipes,
           "source": f"ncu --set full ({os.path.basename(rep)}), summary in r1_ncu_summary.md"},
          open(os.path.join(P, "sense_traffic.json"), "w"), indent=1)
b = json.loads(open(bench).read().strip().splitlines()[-1])
lt = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), "launches",
                     launches], capture_output=True, text=True).stdout
full = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), "full",
                       rep, "c5"], capture_output=True, text=True).stdout
with open(os.path.join(P, "r1_ncu_summary.md"), "a") as f:
    f.write(f"""

## k_sense {tag} (bench c5 {b['ms_per_step']:.4f} ms/step, {b['value']:.3e} agent-steps/s, r1_bench_c5_{tag}.json)

{note}  ncu (cold, serialised): {num('gpu__time_duration.sum')} {rows[1][h.index('gpu__time_duration.sum')]},
{inst / 1e6:.1f} M warp instructions, issue active {num('smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} %,
DRAM {rd:.1f} + {wr:.1f} MB per launch.  Roofline in the bench line: achieved
{b['roofline']['achieved']:.2f} of {b['roofline']['peak']:.2f} (frac {b['roofline']['frac']:.3f}).

Launch list (r1_launches_c5_{tag}.csv):

{lt}
### {tag} full capture

{full}
""")
print("ok", tag, (rd + wr) * unit, inst)
