"""Copy a round-2 evidence run (tools/gpu_round2_evidence.sh -> gpurun_out/) into profiles/:
bench lines, launch lists, parity statistics, slab timing, full-capture metrics, the K4
opcode histogram, sense_traffic.json / stage_traffic.json / stage_traffic_c4.json, and the
summary r2_ncu_summary.md."""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
os.chdir(ROOT)
for a, b in (("bench_c5_r2.json", "r2_bench_c5.json"), ("bench_c4_r2.json", "r2_bench_c4.json"),
             ("launches_c5_r2.csv", "r2_launches_c5.csv"), ("launches_c4_r2.csv", "r2_launches_c4.csv"),
             ("parity_stats_r2.json", "parity_stats.json"), ("slab_timing.json", "r2_slab_timing_1gpu.json"),
             ("launches_slab8_r2.csv", "r2_launches_slab8.csv")):
    shutil.copy(os.path.join(G, a), os.path.join(P, b))

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.per_cycle_active', 'launch__registers_per_thread',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct',
        'launch__grid_size', 'launch__block_size']
m = {}
for f in ("prof_rb_r2b", "prof_k4_r2b", "prof_k7_r2b"):
    raw = subprocess.run(["ncu", "-i", os.path.join(G, f + ".ncu-rep"), "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(raw))
    h, u, d = rows[0], rows[1], dict(zip(rows[0], rows[2]))
    m[f] = {"kernel": d["Kernel Name"][:80]}
    for k in KEYS:
        if k in d:
            m[f][k] = (d[k], u[h.index(k)])
    st = {k: float(v) for k, v in d.items() if "smsp__pcsamp_warps_issue_stalled" in k
          and not k.endswith("not_issued") and v.replace(".", "", 1).isdigit()}
    tot = sum(st.values())
    m[f]["stalls"] = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): round(v / tot * 100, 1)
                      for k, v in sorted(st.items(), key=lambda x: -x[1])[:6]}
json.dump(m, open(os.path.join(G, "r2_full_metrics.json"), "w"), indent=1)
src = subprocess.run(["ncu", "-i", os.path.join(G, "prof_k4_r2b.ncu-rep"), "--page", "source", "--csv",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
open(os.path.join(G, "k4_src_b.csv"), "w").write(src)
subprocess.run([sys.executable, "tools/opcode_hist.py", os.path.join(G, "k4_src_b.csv"), "1e6",
                os.path.join(P, "r2_k4_opcode_hist.md")], capture_output=True, check=True)


def v(f, k):
    return float(m[f][k][0])


def mb(f, k):
    x = m[f][k]
    return float(x[0]) * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3}.get(x[1], 1)


k4 = "prof_k4_r2b"
json.dump({"config": "c5", "kernel": m[k4]["kernel"].split("(")[0] + " (round 2)",
           "bytes_per_launch": mb(k4, "dram__bytes_read.sum") + mb(k4, "dram__bytes_write.sum"),
           "dram_read_bytes": mb(k4, "dram__bytes_read.sum"), "dram_write_bytes": mb(k4, "dram__bytes_write.sum"),
           "warp_instructions": v(k4, "smsp__inst_executed.sum"), "candidate_tests": None,
           "pct_of_peak": {"issue_active": v(k4, "smsp__issue_active.avg.pct_of_peak_sustained_active")},
           "source": "ncu --set full (gpurun_out/prof_k4_r2b.ncu-rep), summary in r2_ncu_summary.md"},
          open(os.path.join(P, "sense_traffic.json"), "w"), indent=1)
rb = "prof_rb_r2b"
json.dump({"config": "c4", "kernel": "void k_replica_bin<0, 1, 1> (MODE 1: persistent, shared-memory staged)",
           "dram_read_B": int(mb(rb, "dram__bytes_read.sum")), "dram_write_B": int(mb(rb, "dram__bytes_write.sum")),
           "ncu_us": v(rb, "gpu__time_duration.sum"), "alg_bytes": 92 * 5120000,
           "source": "ncu --set full --clock-control none (gpurun_out/prof_rb_r2b.ncu-rep; cold caches, one launch)"},
          open(os.path.join(P, "stage_traffic_c4.json"), "w"), indent=1)
rows = [r for r in csv.reader(open(os.path.join(G, "launches_c5_r2.csv"))) if len(r) > 5]
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[1:]:
    val = float(r[vi].replace(",", ""))
    val *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[ui], 1)
    if r[ui] == "ns":
        val /= 1e3
    agg[r[ki].split("(")[0]][r[mi]].append(val)
mean = lambda k, mm: sum(agg[k][mm]) / len(agg[k][mm])  # noqa: E731
names = sorted(agg)
pick = lambda pre: next(n for n in names if n.startswith(pre))  # noqa: E731
mp = {"integrate_bin": [pick("void vg::k_integrate_bin<0, 1, 1>")],
      "scan_cells": [pick("vg::k_scan_tiles"), pick("vg::k_scan_apply")],
      "scatter": [pick("void vg::k_scatter<0>")], "cell_sort": [pick("vg::k_cell_sort")],
      "sense": [pick("void vg::k_sense<0, 1, 0, 0, 2")]}
json.dump({"config": "c5", "source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                                     "(cold caches, serialised launches; round-2 kernels; profiles/r2_launches_c5.csv)",
           "stages": {st: {"dram_read_B": int(sum(mean(k, "dram__bytes_read.sum") for k in ks)),
                           "dram_write_B": int(sum(mean(k, "dram__bytes_write.sum") for k in ks)),
                           "ncu_us": round(sum(mean(k, "gpu__time_duration.sum") for k in ks), 3),
                           "kernels": [k.replace("vg::", "") for k in ks]} for st, ks in mp.items()}},
          open(os.path.join(P, "stage_traffic.json"), "w"), indent=1)
print("profiles refreshed")
