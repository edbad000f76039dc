"""Summarise `ncu --page source --csv --print-source sass`: instruction mix
(executed warp instructions by opcode) and the top stall-sampled lines.

    python tools/sass_hot.py gpurun_out/src.csv [top]
"""
import collections
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(path)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
mix = collections.Counter()
samples = []
total = 0
for r in rows[2:]:
    if len(r) < len(hdr) or not r[ix["Address"]].startswith("0x"):
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    n = int(r[ix["Instructions Executed"]] or 0)
    mix[op.split(".")[0]] += n
    total += n
    samples.append((int(r[ix["Warp Stall Sampling (All Samples)"]] or 0), src, n))
print(f"total warp instructions: {total:,}")
for op, n in mix.most_common(30):
    print(f"  {op:10s} {n:14,d} {n / total:6.1%}")
print("top stall-sampled instructions:")
for s, src, n in sorted(samples, reverse=True)[:top]:
    print(f"  {s:6d}  {src[:80]}")

# stall reasons: totals over the kernel, and for the top instructions
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {r: 0 for r in reasons}
per = []
for r in rows[2:]:
    if len(r) < len(hdr) or not r[ix["Address"]].startswith("0x"):
        continue
    vals = {k: int(r[ix[k]] or 0) for k in reasons}
    for k in reasons:
        tot[k] += vals[k]
    per.append((sum(vals.values()), r[ix["Source"]].strip(), vals))
allv = sum(tot.values()) or 1
print("stall reasons (share of samples):")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {k:22s} {v / allv:6.1%}")
print("top instructions by samples, with their main reasons:")
for s, src, vals in sorted(per, key=lambda t: -t[0])[:top]:
    main = ", ".join(f"{k[6:]}={v}" for k, v in sorted(vals.items(), key=lambda kv: -kv[1])[:3] if v)
    print(f"  {s:6d}  {src[:48]:48s} {main}")
