"""Turn raw ncu / bench outputs (gpurun_out/) into the committed evidence in profiles/.

    python tools/collect_profiles.py --round 1

* launches_<w>.csv  (ncu --metrics gpu__time_duration.sum,dram__bytes_*)
    -> profiles/r<NN>_launches_<w>.txt : per kernel, median device time and
       DRAM bytes per launch, and its share of the listed time
* ncu_details_<tag>.csv / ncu_raw_<tag>.csv (ncu --set full)
    -> profiles/r<NN>_ncu_<tag>.txt : key throughput / occupancy / stall metrics
* profiles/ncu_traffic.json : "<workload>:<op>" -> dram bytes per launch of the
  op's kernel (bench.py reads it for roofline.traffic)
* bench.json -> profiles/r<NN>_bench_<w>.json
"""

import argparse
import collections
import csv
import glob
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from ncu_summary import summarise  # noqa: E402

OP_KERNELS = {  # bench op -> kernel name prefix
    "compress": ("k_dct8_compress", "k_dct4_compress", "k_fast_compress", "k_half3_compress",
                 "k_exact_compress"),
    "decompress": ("k_dct8_decompress", "k_dct4_decompress", "k_fast_decompress", "k_half3_decompress",
                   "k_exact_decompress"),
    "l2_norm": ("k_moments_stream", "k_moments_staged"),  # PAIR = false instantiation
    "dot": ("k_moments_stream", "k_moments_staged"),      # PAIR = true
    "add": ("k_add8", "k_add_small", "k_add", "k_add_staged", "k_add_tiled"),
}

STALL_KEYS = [
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "smsp__inst_executed.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {h: i for i, h in enumerate(hdr)}
    data = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        name = r[ix["Kernel Name"]].split("(")[0]
        try:
            data[name][r[ix["Metric Name"]]].append(float(r[ix["Metric Value"]].replace(",", "")))
        except ValueError:
            pass
    return data


def raw_stalls(path):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return []
    hdr = rows[0]
    out = []
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        name = r[hdr.index("Kernel Name")].split("(")[0]
        vals = {k: r[hdr.index(k)] for k in STALL_KEYS if k in hdr}
        out.append((name, vals))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", type=int, default=1)
    ap.add_argument("--src", default=os.path.join(ROOT, "gpurun_out"))
    args = ap.parse_args()
    tag = f"r{args.round:02d}"
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    traffic_path = os.path.join(prof, "ncu_traffic.json")
    old = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    traffic = {}  # rebuilt from this round's launch lists; workloads not profiled keep old values

    for path in sorted(glob.glob(os.path.join(args.src, "launches_*.csv"))):
        w = os.path.basename(path)[len("launches_"):-4]
        data = launches(path)
        total = sum(statistics.median(m["gpu__time_duration.sum"]) * len(m["gpu__time_duration.sum"])
                    for m in data.values() if m.get("gpu__time_duration.sum"))
        lines = [f"# ncu launch list, workload {w} (tools/profile_ops.py; cold-cache, serialised)",
                 f"# {'kernel':58s} {'launches':>8s} {'median_us':>10s} {'dram_MB':>9s} {'share':>6s}"]
        for name, m in sorted(data.items(), key=lambda kv: -sum(kv[1].get("gpu__time_duration.sum", [0]))):
            t = m.get("gpu__time_duration.sum", [])
            if not t:
                continue
            dram = [a + b for a, b in zip(m.get("dram__bytes_read.sum", []), m.get("dram__bytes_write.sum", []))]
            med = statistics.median(t)
            share = med * len(t) / total if total else 0
            lines.append(f"{name[:58]:58s} {len(t):8d} {med / 1e3:10.1f} "
                         f"{(statistics.median(dram) / 1e6 if dram else 0):9.1f} {share:6.3f}")
            for op, prefixes in OP_KERNELS.items():
                targs = name[name.find("<") + 1:name.rfind(">")].split(", ") if "<" in name else []
                if op in ("l2_norm", "dot") and "moments_stream" in name:
                    pair = len(targs) > 3 and targs[3] in ("1", "true")
                    if pair != (op == "dot"):
                        continue
                if op == "decompress" and targs and "double" not in targs:
                    continue  # bench "decompress" is the f64-output call
                base = name.split("<")[0].split("::")[-1].split()[-1]
                if any(base == p or base.startswith(p + "_") for p in prefixes) and dram:
                    key = f"{w}:{op}"
                    if "to_kind" not in key and key not in traffic:  # dominant kernel first
                        traffic[key] = statistics.median(dram)
        with open(os.path.join(prof, f"{tag}_launches_{w}.txt"), "w") as fh:
            fh.write("\n".join(lines) + "\n")

    for path in sorted(glob.glob(os.path.join(args.src, "ncu_details_*.csv"))):
        t = os.path.basename(path)[len("ncu_details_"):-4]
        text = summarise(path)
        raw = os.path.join(args.src, f"ncu_raw_{t}.csv")
        if os.path.exists(raw):
            text += "\n\n# stall reasons / pipes / traffic (raw page)\n"
            for name, vals in raw_stalls(raw):
                text += name + "\n" + "".join(f"    {k} = {v}\n" for k, v in vals.items())
        with open(os.path.join(prof, f"{tag}_ncu_{t}.txt"), "w") as fh:
            fh.write(text + "\n")

    bench = os.path.join(args.src, "bench.json")
    if os.path.exists(bench):
        lines = [l for l in open(bench) if l.strip().startswith("{")]
        if lines:
            d = json.loads(lines[-1])
            w = "c2" if "C2" in d.get("config", {}).get("workload", "") else "x"
            with open(os.path.join(prof, f"{tag}_bench_{w}.json"), "w") as fh:
                json.dump(d, fh, indent=1)
    for k, v in old.items():
        traffic.setdefault(k, v)
    with open(traffic_path, "w") as fh:
        json.dump(traffic, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
