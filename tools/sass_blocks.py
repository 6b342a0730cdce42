"""Group an ncu SASS source page (--page source --csv --print-source sass) into straight-line
blocks by execution count and print the heaviest ones (per-agent warp instructions)."""
import csv
import sys

path, agents = sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1e6
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if "Address" in r and "Source" in r][0]
hdr, data = rows[hi], rows[hi + 1:]
ia, isrc = hdr.index("Instructions Executed"), hdr.index("Source")
ins = [(r[isrc].strip(), int(r[ia])) for r in data if len(r) > ia and r[ia].isdigit()]
print("total warp instructions", sum(n for _, n in ins), "per agent", sum(n for _, n in ins) / agents)
blocks, cur = [], None
for k, (s, n) in enumerate(ins):
    if cur and cur[1] == n:
        cur[2].append(s)
    else:
        cur = [k, n, [s]]
        blocks.append(cur)
blocks.sort(key=lambda b: -b[1] * len(b[2]))
for k, n, l in blocks[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]:
    print(f"{k:5d} n={n:9d} len={len(l):3d} per_agent={n * len(l) / agents:7.1f} :: " +
          " | ".join(x[:24] for x in l[:4]))
