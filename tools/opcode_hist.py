"""Executed-instruction histogram by SASS opcode from an ncu source page export
(`ncu -i rep --page source --csv --print-source sass -k <kernel>`): warp instructions per
agent per opcode (and per opcode family), for profiles/ (K4 instruction diet).

Usage: python tools/opcode_hist.py source.csv n_agents [out.md]"""
import collections
import csv
import re
import sys

path, agents = sys.argv[1], float(sys.argv[2])
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if "Source" in r and any("Instructions Executed" in c for c in r)][0]
hdr, data = rows[hi], rows[hi + 1:]
ie = [i for i, c in enumerate(hdr) if c.strip() == "Instructions Executed"][0]
isrc = hdr.index("Source")
ops, fam = collections.Counter(), collections.Counter()
total = 0
for r in data:
    if len(r) <= max(ie, isrc) or not r[ie].strip().isdigit():
        continue
    n = int(r[ie])
    s = re.sub(r"^@!?U?P\w+\s+", "", r[isrc].strip())
    op = s.split(" ")[0].rstrip(";")
    if not op:
        continue
    ops[op] += n
    fam[op.split(".")[0]] += n
    total += n
out = [f"total warp instructions {total} = {total / agents:.1f} per agent", "",
       "| opcode family | warp instr / agent | share |", "|---|---|---|"]
for k, v in fam.most_common():
    if v / agents >= 0.5:
        out.append(f"| {k} | {v / agents:.1f} | {v / total:.3f} |")
out += ["", "| opcode | warp instr / agent |", "|---|---|"]
for k, v in ops.most_common(40):
    out.append(f"| `{k}` | {v / agents:.1f} |")
text = "\n".join(out)
print(text)
if len(sys.argv) > 3:
    open(sys.argv[3], "w").write(text + "\n")
