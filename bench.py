"""Benchmark driver: the PyBlaz hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c1|c3|c5]

Default workload = BASELINE.json configs[1] (C2): a 2-D float64 8192x8192
array per GPU, 4x4 blocks, int16 indices, F64 maxima, full mask.  One step =
compress -> L2 norm -> decompress (float64 out) through the public API's
kernels.  N > 1 (torchrun, one process per GPU, NCCL): the array is
block-row sharded, 8192 rows per GPU (weak scaling); the L2 norm all-gathers
the shards' partial records over NCCL -- the only cross-GPU traffic.

`value` = uncompressed input GB/s of the whole job (all ranks) with inputs
resident in HBM (> L2, so no flush needed), max over ranks of CUDA-event time.
`e2e` = the same step through the public API from pinned HOST memory,
including the H2D copy of the input and the D2H copy of the decompressed
result every step.  `--impl reference` times the CPU oracle port
(oracle/bzc_oracle.py, numpy; the reference is pure Python and cannot travel
to the GPU box) on all host cores, one process per core over block-row slabs.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "compress/decompress GB/s and compressed dot/L2 GB/s vs HBM roofline, 1/2/4/8 GPU"

WORKLOADS = {
    # name: (per-GPU shape, block, float kind, index kind, lowpass mask, description)
    "c2": ((8192, 8192), (4, 4), "f64", "i16", None,
           "C2: 2-D float64 8192x8192 per GPU, block 4x4, int16 index, F64 maxima, full mask; "
           "step = compress + L2 norm + decompress (f64 out)"),
    "c1": ((256, 256, 256), (8, 8, 8), "f32", "i8", None,
           "C1: 3-D float32 256^3, block 8x8x8, int8 index, F32 maxima, full mask; "
           "step = compress + L2 norm + decompress (f64 out)"),
    "c3": ((1024, 1024, 1024), (8, 8, 8), "f32", "i8", None,
           "C3: 3-D float32 1024^3 per GPU, block 8x8x8, int8 index; step = compress + L2 norm "
           "+ decompress (f64 out)"),
    "c5": ((256, 256, 256, 64), (4, 4, 4, 4), "f32", "i8", 4,
           "C5: 4-D float32 (256,256,256,64), block 4^4, int8 index, low-pass mask "
           "(sum idx <= 4, K=66); step = compress + L2 norm + decompress (f64 out)"),
}


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def load_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def load_traffic():
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except Exception:
        return {}


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML every
    ~2 ms while the benchmark runs (warm-up and timed region)."""

    def __init__(self, torch_device):
        self.dev = torch_device
        self.samples = []          # (t, sm_mhz, reasons_bitmask)
        self.t0 = self.t1 = None
        self._stop = threading.Event()
        self.handle = None
        self.max_mhz = None

    def _open(self):
        import pynvml
        import torch

        pynvml.nvmlInit()
        props = torch.cuda.get_device_properties(self.dev)
        handle = None
        uuid = getattr(props, "uuid", None)
        if uuid is not None:
            try:
                handle = pynvml.nvmlDeviceGetHandleByUUID("GPU-" + str(uuid))
            except Exception:
                handle = None
        if handle is None:
            handle = pynvml.nvmlDeviceGetHandleByIndex(self.dev.index or 0)
        self.handle = handle
        self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(handle, pynvml.NVML_CLOCK_SM)

    def _run(self):
        import pynvml

        while not self._stop.is_set():
            try:
                mhz = pynvml.nvmlDeviceGetClockInfo(self.handle, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
                self.samples.append((time.perf_counter(), mhz, rs))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        try:
            self._open()
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception:
            self.handle = None
        return self

    def mark(self, start: bool):
        if start:
            self.t0 = time.perf_counter()
        else:
            self.t1 = time.perf_counter()

    def __exit__(self, *exc):
        self._stop.set()
        if self.handle is not None:
            self.thread.join(timeout=2)

    def summary(self):
        import pynvml

        names = {
            "hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
            "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
            "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
            "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap,
            "hw_power_brake": pynvml.nvmlClocksEventReasonHwPowerBrakeSlowdown,
        }
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        timed = [s for s in self.samples
                 if self.t0 is not None and self.t1 is not None and self.t0 <= s[0] <= self.t1]
        use = timed if timed else self.samples
        mhz = [s[1] for s in use]
        reasons = sorted({n for n, bit in names.items() for s in use if s[2] & bit})
        return {"sm_mhz": statistics.median(mhz), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(use),
                "window": "timed region" if timed else "warm-up + timed region (region < 2 ms)"}


# --------------------------------------------------------------------- ours --
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2406_11209_b200 as bz
    from paper_2406_11209_b200 import _native
    from paper_2406_11209_b200 import distributed as bd
    from paper_2406_11209_b200.ops import merge_records, moments_record, Record

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        world = args.gpus if world == 1 and args.gpus == 1 else world
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    shape, block, fk, ik, lowpass, desc = WORKLOADS[args.workload]
    kind = bz.FloatKind(fk)
    mask = None
    if lowpass is not None:
        mask = bz.PruningMask(block, np.indices(block).sum(axis=0) <= lowpass)
    s = bz.CodecSettings(block, kind, bz.IndexKind(ik), bz.TransformFamily.DCT, mask)
    global_shape = (shape[0] * world,) + tuple(shape[1:])
    n_local = int(np.prod(shape))
    in_bytes_local = n_local * kind.itemsize
    B = int(np.prod(s.grid_for(shape)))
    K = s.mask.kept_count
    comp_bytes = B * (K * s.index_kind.itemsize + kind.itemsize)

    # synthetic input, counter-based and partition invariant (global flat offset)
    x = torch.empty(shape, dtype=kind.torch_dtype, device=dev)
    _native.call("bz_fill_random", x.data_ptr(), kind.code, n_local, rank * n_local, 2, 0,
                 _native.stream_handle(dev))
    xa = bz.DenseArray.wrap(x, kind)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def gather(rec):
        if world == 1:
            return [rec]
        out = [torch.empty_like(rec) for _ in range(world)]
        dist.all_gather(out, rec)
        return out

    records = []

    def step():
        ca = bz.compress(xa, s)
        recs = gather(moments_record(ca, dc_only=2))  # "sums": what l2_norm uses
        out = bz.decompress(ca)
        records.append(recs)
        return out

    def timed(fn, reps):
        barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        return max_over_ranks(e0.elapsed_time(e1) / reps)

    # ---- warmup + timed steps (device-resident inputs); clocks sampled throughout
    with ClockSampler(dev) as clocks:
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize(dev)
        records.clear()
        launches0 = _native.query("bz_launch_count")
        clocks.mark(True)
        ms_step = timed(step, args.steps)
        clocks.mark(False)
        launches = _native.query("bz_launch_count") - launches0
    # the L2 norms of the timed steps (host epilogue after the timed region)
    l2_vals = []
    for recs in records:
        r = merge_records([Record.from_array(t.cpu().numpy()) for t in recs])
        l2_vals.append(math.sqrt(max(r.s_aa + r.m_aa + r.n * r.mean_a ** 2, 0.0))
                       / s.index_kind.radius)
    value = world * in_bytes_local / (ms_step * 1e-3) / 1e9

    # ---- per-op breakdown (same kernels, timed one by one)
    ca = bz.compress(xa, s)
    reps = max(args.steps, 5)
    ops = {}
    peak, peak_src = load_peak()

    def op(name, fn, alg_bytes, in_bytes):
        for _ in range(3):
            fn()
        ms = timed(fn, reps)
        ops[name] = {"ms": round(ms, 5), "gbs_uncompressed": round(in_bytes / ms / 1e6, 1),
                     "gbs_algorithmic": round(alg_bytes / ms / 1e6, 1),
                     "roofline_frac": round(alg_bytes / ms / 1e6 / peak, 4),
                     "alg_bytes": alg_bytes}

    op("compress", lambda: bz.compress(xa, s), in_bytes_local + comp_bytes, in_bytes_local)
    op("l2_norm", lambda: gather(moments_record(ca, dc_only=2)), comp_bytes, in_bytes_local)
    op("decompress", lambda: bz.decompress(ca), comp_bytes + n_local * 8, in_bytes_local)
    op("decompress_to_kind", lambda: bz.decompress(ca, kind), comp_bytes + n_local * kind.itemsize,
       in_bytes_local)
    cb = bz.compress(bz.DenseArray.wrap(torch.flip(x, dims=[0]).contiguous(), kind), s)
    op("dot", lambda: gather(moments_record(ca, cb, dc_only=2)), 2 * comp_bytes, 2 * in_bytes_local)
    dominant = max(("compress", "decompress"), key=lambda k: ops[k]["ms"])
    traffic = load_traffic().get(f"{args.workload}:{dominant}")
    roofline = {
        "kernel": dominant,
        "bound": "hbm",
        "achieved": ops[dominant]["gbs_algorithmic"],
        "peak": peak,
        "unit": "GB/s",
        "frac": ops[dominant]["roofline_frac"],
        "traffic": traffic,
        "peak_source": peak_src,
        "alg_bytes_per_launch": ops[dominant]["alg_bytes"],
    }

    # ---- end to end through the public API from pinned host memory.  Steps
    #      alternate between two CUDA streams, so step i's D2H copy of the
    #      decompressed array overlaps step i+1's H2D copy (PCIe is full duplex);
    #      every step still pays its own H2D, D2H and the scalar read-back.
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    host_in = [torch.empty(shape, dtype=kind.torch_dtype, pin_memory=True) for _ in streams]
    for h in host_in:
        h.copy_(x.cpu())
    host_out = [torch.empty(shape, dtype=torch.float64, pin_memory=True) for _ in streams]
    e2e_l2 = []
    e2e_i = [0]

    def e2e_step():
        i = e2e_i[0] % 2
        e2e_i[0] += 1
        st = streams[i]
        with torch.cuda.stream(st):
            a = bz.DenseArray(shape, kind, host_in[i])       # H2D copy (async, pinned)
            c = bz.compress(a, s)
            if world == 1:
                e2e_l2.append(bz.l2_norm(c))                 # D2H of the scalar (syncs st)
            else:
                e2e_l2.append(bz.l2_norm(bd.ShardedCompressedArray(c, global_shape)))
            out = bz.decompress(c)
            host_out[i].copy_(out.values, non_blocking=True)  # D2H copy of the result

    def e2e_timed(reps):
        barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for st in streams:
            st.wait_event(e0)
        for _ in range(reps):
            e2e_step()
        for st in streams:
            stream.wait_stream(st)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        return max_over_ranks(e0.elapsed_time(e1) / reps)

    e2e_steps = max(8, args.steps // 2)  # steady state: first H2D and last D2H are not overlapped
    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize(dev)
    ms_e2e = e2e_timed(e2e_steps)
    e2e = {
        "value": round(world * in_bytes_local / (ms_e2e * 1e-3) / 1e9, 3),
        "unit": "GB/s",
        "h2d_bytes_per_step": in_bytes_local,
        "d2h_bytes_per_step": n_local * 8 + 8,
        "ms_per_step": round(ms_e2e, 4),
        "steps": e2e_steps,
        "path": "DenseArray(pinned host) -> compress -> l2_norm (float) -> decompress -> "
                "host copy; two streams alternate so D2H of step i overlaps H2D of step i+1",
    }

    result = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(args.workload)
        result = {
            "metric": METRIC,
            "value": round(value, 3),
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_step, 5),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": fk,
            "data": "synthetic: counter-based N(0,1), partition-invariant (bz_fill_random)",
            "config": {
                "workload": desc,
                "global_shape": list(global_shape),
                "per_gpu_shape": list(shape),
                "block": list(block),
                "float_kind": fk,
                "index_kind": ik,
                "kept": K,
                "parallelism": f"block-row shards x{world}, NCCL all_gather of partial records",
                "l2_flush": f"not needed: inputs are {in_bytes_local / 2**20:.0f} MiB per GPU > 126 MB L2",
                "fast_path": bz.is_fast_path(s, shape),
            },
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
            "ops": ops,
            "l2_norm_check": {"min": min(l2_vals), "max": max(l2_vals)},
        }
        print(json.dumps(result))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return result


# ---------------------------------------------------------------- CPU side --
def _oracle_settings(workload):
    import numpy as np

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import bzc_oracle as o

    shape, block, fk, ik, lowpass, _ = WORKLOADS[workload]
    bits = None if lowpass is None else (np.indices(block).sum(axis=0) <= lowpass)
    return o, o.Settings(block, fk, ik, "dct", bits)


def _slab(workload, rows, seed):
    import numpy as np

    shape, block, fk, *_ = WORKLOADS[workload]
    rng = np.random.default_rng(seed)
    o, _s = _oracle_settings(workload)
    return o.round_to_kind(rng.normal(size=(rows,) + tuple(shape[1:])), fk)


def _cpu_step(o, s, x):
    c = o.compress(x, s)
    k = s.kept
    p = c.indices.reshape(-1, k).astype("float64") * c.maxima.reshape(-1, 1)
    sq = float((p * p).sum())
    o.decompress(c)
    return sq


def cpu_baseline(workload, min_seconds=10.0, max_reps=20):
    """The oracle port on ONE core (BLAS pinned to one thread), bounded sample."""
    try:
        from threadpoolctl import threadpool_limits
    except Exception:  # pragma: no cover
        threadpool_limits = None
    shape, block, fk, *_ = WORKLOADS[workload]
    rows = max(block[0], shape[0] // 8 // block[0] * block[0])
    o, s = _oracle_settings(workload)
    x = _slab(workload, rows, 2)
    nbytes = x.size * (8 if fk == "f64" else 4)
    ctx = threadpool_limits(limits=1) if threadpool_limits else None
    if ctx:
        ctx.__enter__()
    try:
        _cpu_step(o, s, x)
        times = []
        t_all = time.perf_counter()
        while len(times) < max_reps and (time.perf_counter() - t_all) < min_seconds:
            t0 = time.perf_counter()
            _cpu_step(o, s, x)
            times.append(time.perf_counter() - t0)
    finally:
        if ctx:
            ctx.__exit__(None, None, None)
    t = statistics.median(times)
    return {
        "value": round(nbytes / t / 1e9, 4),
        "unit": "GB/s",
        "cores": 1,
        "kind": "port",
        "sample": f"{rows}x{'x'.join(map(str, shape[1:]))} slab ({x.size} elements, 1/8 of one "
                  f"GPU's array); step = compress + L2 + decompress; median of {len(times)} "
                  f"reps ({t:.3f} s each); numpy oracle, BLAS 1 thread",
    }


_W = {}


def _ref_init(workload, rows, seed):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    o, s = _oracle_settings(workload)
    _W["o"], _W["s"] = o, s
    _W["x"] = _slab(workload, rows, seed)


def _ref_task(_):
    return _cpu_step(_W["o"], _W["s"], _W["x"])


def run_reference(args):
    rank = env_int("RANK", 0)
    if rank != 0:
        return None
    import multiprocessing as mp

    shape, block, fk, ik, lowpass, desc = WORKLOADS[args.workload]
    procs = max(1, os.cpu_count() or 1)
    # size the per-step sample so one step takes ~2 s on this host
    per_row_1core = 0.8e-3 * (shape[1] if len(shape) > 1 else 1) / 8192 * \
        (int(__import__("numpy").prod(shape[2:])) if len(shape) > 2 else 1)
    rows_total = int(min(shape[0], max(block[0], 2.0 * procs / max(per_row_1core, 1e-9))))
    rows_per = max(block[0], (rows_total // procs) // block[0] * block[0])
    procs = max(1, min(procs, rows_total // rows_per))
    rows_total = rows_per * procs
    ctx = mp.get_context("spawn")
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    pools = [ctx.Pool(1, initializer=_ref_init, initargs=(args.workload, rows_per, 100 + i))
             for i in range(procs)]
    try:
        def one_step():
            res = [p.apply_async(_ref_task, (0,)) for p in pools]
            return sum(r.get() for r in res)

        for _ in range(max(1, args.warmup)):
            one_step()
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            one_step()
            times.append(time.perf_counter() - t0)
    finally:
        for p in pools:
            p.close()
            p.join()
    elem = rows_total * int(__import__("numpy").prod(shape[1:]))
    nbytes = elem * (8 if fk == "f64" else 4)
    t = statistics.mean(times)
    value = nbytes / t / 1e9
    sample = (f"{rows_total}x{'x'.join(map(str, shape[1:]))} per step ({rows_per} rows per "
              f"process x {procs} processes); step = compress + L2 + decompress")
    out = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(value, 4),
        "unit": "GB/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(t * 1e3, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": fk,
        "data": "synthetic: numpy N(0,1)",
        "config": {"workload": desc, "per_gpu_shape": list(shape), "block": list(block),
                   "float_kind": fk, "index_kind": ik},
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": procs, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", choices=sorted(WORKLOADS), default="c2")
    p.add_argument("--no-cpu-baseline", action="store_true")
    args = p.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
