"""Per-kernel registers / spills from `nvcc -Xptxas -v` output (stdin): one line per entry."""
import re
import subprocess
import sys

txt = sys.stdin.read()
cur = None
rows = {}
for line in txt.splitlines():
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = m.group(1)
        rows[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        rows[cur]["spill"] = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows[cur]["regs"] = int(m.group(1))
names = subprocess.run(["c++filt"], input="\n".join(rows), capture_output=True, text=True).stdout.split("\n")
pat = sys.argv[1] if len(sys.argv) > 1 else ""
for (k, v), n in zip(rows.items(), names):
    if pat in n:
        short = re.sub(r"\(.*", "", n)
        print(f"{short:50s} regs={v.get('regs')} spill={v.get('spill')}")
