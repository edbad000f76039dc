"""Walk the SASS of one kernel (ncu source page CSV) in address order and
print executed warp instructions per opcode for each region between
markers (shared-memory ops / syncs), to attribute instruction counts to
the phases of the kernel.

    python tools/sass_regions.py gpurun_out/src_x.csv [min_count]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
mincnt = int(sys.argv[2]) if len(sys.argv) > 2 else 1
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
seq = []
for r in rows[2:]:
    if len(r) < len(hdr) or not r[ix["Address"]].startswith("0x"):
        continue
    src = r[ix["Source"]].strip()
    n = int(r[ix["Instructions Executed"]] or 0)
    op = src.split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    seq.append((int(r[ix["Address"]], 16), o, n, src))
total = sum(n for _, _, n, _ in seq)
print(f"total {total:,}")
# segment: a new region starts at every WARPSYNC / BAR / first STS after LDS etc.
region = collections.Counter()
start = None
cnt = 0
def flush(tag):
    global region, cnt
    if cnt:
        top = ", ".join(f"{k.split('.')[0]} {v/1e6:.1f}" for k, v in region.most_common(8))
        print(f"{tag:>12} {cnt/1e6:8.1f}M  {top}")
    region = collections.Counter()
    cnt = 0
for a, o, n, src in seq:
    if n < mincnt:
        continue
    if o.startswith("WARPSYNC") or o.startswith("BAR") or o.startswith("NOP"):
        flush(hex(a))
        continue
    region[o.split('.')[0]] += n
    cnt += n
flush("end")
