"""Summarise an `ncu --page details --csv` export: one line of key metrics per kernel."""
import csv
import collections
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Issue Slots Busy", "Executed Ipc Active", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size", "SM Frequency"]


def summarise(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    per = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) < 15:
            continue
        k = (r[ix["ID"]], r[ix["Kernel Name"]].split("(")[0])
        per.setdefault(k, {})[r[ix["Metric Name"]]] = (r[ix["Metric Value"]], r[ix["Metric Unit"]])
    out = []
    for (kid, name), m in per.items():
        out.append(f"[{kid}] {name}\n    " + "; ".join(
            f"{n}={m[n][0]}{m[n][1]}" for n in WANT if n in m))
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        print(summarise(p))


def traffic_from_raw(path):
    """{kernel name: dram bytes (read+write) per launch, median over launches}."""
    import statistics

    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    rd = ix.get("dram__bytes_read.sum")
    wr = ix.get("dram__bytes_write.sum")
    per = collections.defaultdict(list)
    for r in rows[2:]:  # row 1 holds units
        if len(r) < len(hdr) or rd is None:
            continue
        try:
            per[r[ix["Kernel Name"]].split("(")[0]].append(
                float(r[rd].replace(",", "")) + float(r[wr].replace(",", "")))
        except ValueError:
            continue
    return {k: statistics.median(v) for k, v in per.items()}
