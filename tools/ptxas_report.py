"""Summarise `nvcc -Xptxas -v` output: one line per kernel (regs, stack, spills).

    nvcc ... -Xptxas -v -c file.cu 2>&1 | python tools/ptxas_report.py [name-filter]
"""
import re
import subprocess
import sys

flt = sys.argv[1] if len(sys.argv) > 1 else ""
cur = None
rows = {}
for line in sys.stdin:
    m = re.search(r"Function properties for (\w+)", line)
    if m:
        cur = m.group(1)
        rows.setdefault(cur, {})
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        rows[cur]["stack"], rows[cur]["spill_st"], rows[cur]["spill_ld"] = m.groups()
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows[cur]["regs"] = m.group(1)
names = list(rows)
dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
for n, d in zip(names, dem):
    if flt in d:
        r = rows[n]
        print(f"{r.get('regs','?'):>4} regs stack {r.get('stack','?'):>4} spill {r.get('spill_st','?')}/{r.get('spill_ld','?')}  {d[:110]}")
