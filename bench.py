"""Benchmark driver: the PyBlaz hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c1|c3|c4|c5] [--scaling weak|strong] [--dry-run]

Workloads (BASELINE.json configs; one step = one pass of the path):

* c2 (default; configs[1], the single-B200 config the metric is quoted on):
  2-D float64 8192x8192 per GPU, 4x4 blocks, int16 indices; step = compress
  -> L2 norm -> decompress (f64 out).  Weak scaling: 8192 rows per GPU.
* c1: configs[0] shape (256^3 f32, 8^3, int8), same step; weak.
* c3: configs[2], 1024^3 f32 8^3 int8: compress(x) -> add(x, y) ->
  mul_scalar(0.5) -> mean + variance (one fused pass).  Strong scaling.
* c4: configs[3], two 1024^3 f32 fields: compress both -> covariance, cosine
  similarity and SSIM from ONE fused pair pass.  Strong scaling.
* c5: configs[4], 4-D (256,256,256,64) f32 4^4 int8, low-pass mask (K=66):
  compress(x_t) -> fused l2(x_t - x_{t-1}) -> decompress.  Strong scaling.

Multi-GPU: ``--gpus N`` without a torchrun environment re-launches itself
under ``torch.distributed.run`` (one process per GPU, NCCL, 127.0.0.1).
The block grid is split along axis 0 into contiguous block-row shards
(strong: the global shape is fixed; weak: each GPU holds the per-GPU shape);
compress / decompress / elementwise ops are shard-local, each reduction is
ONE all_gather_into_tensor of the ranks' 16-double records (the only
cross-GPU traffic).  Times are CUDA-event times, max over ranks.

`value` = uncompressed input GB/s of the whole job with inputs resident in
HBM (> L2, so no flush is needed).  `e2e` = the same step through the public
API from pinned HOST memory (H2D of the input and D2H of the result inside
the timed region).  `cpu_baseline` (rank 0, N=1): the reference package
``bzc`` from ``baseline/_ref`` on one core over a bounded slab (the numpy
oracle port when the install is absent, labelled "port"); the same slab is
run through the GPU path and compared with the reference's outputs
(``parity``: index mismatches, rounding-tie fraction, decompression and
operator relative errors).  ``--impl reference`` times the reference package
on all host cores (one process per core over block-row slabs).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "compress/decompress GB/s and compressed dot/L2 GB/s vs HBM roofline, 1/2/4/8 GPU"

WORKLOADS = {
    # name: shape (per GPU for weak, global for strong), block, float kind,
    #       index kind, low-pass mask order (None = full), default scaling, step, description
    "c2": dict(shape=(8192, 8192), block=(4, 4), fk="f64", ik="i16", lowpass=None,
               scaling="weak", step="codec",
               desc="C2: 2-D float64 8192x8192 per GPU, block 4x4, int16 index, F64 maxima, "
                    "full mask; step = compress + L2 norm + decompress (f64 out)"),
    "c1": dict(shape=(256, 256, 256), block=(8, 8, 8), fk="f32", ik="i8", lowpass=None,
               scaling="weak", step="codec",
               desc="C1: 3-D float32 256^3 per GPU, block 8x8x8, int8 index, full mask; "
                    "step = compress + L2 norm + decompress (f64 out)"),
    "c3": dict(shape=(1024, 1024, 1024), block=(8, 8, 8), fk="f32", ik="i8", lowpass=None,
               scaling="strong", step="chain",
               desc="C3: 3-D float32 1024^3, block 8x8x8, int8 index; step = compress(x) + "
                    "add(x, y) + mul_scalar(0.5) + mean/variance (one fused pass)"),
    "c4": dict(shape=(1024, 1024, 1024), block=(8, 8, 8), fk="f32", ik="i8", lowpass=None,
               scaling="strong", step="pair",
               desc="C4: two 3-D float32 1024^3 fields, block 8x8x8, int8 index; step = "
                    "compress both + covariance, cosine similarity, SSIM (one fused pair pass)"),
    "c5": dict(shape=(256, 256, 256, 64), block=(4, 4, 4, 4), fk="f32", ik="i8", lowpass=4,
               scaling="strong", step="sweep",
               desc="C5: 4-D float32 (256,256,256,64), block 4^4, int8 index, low-pass mask "
                    "(sum idx <= 4, K=66); step = compress(x_t) + l2(x_t - x_{t-1}) (fused) + "
                    "decompress (f64 out)"),
}

ITEMSIZE = {"f64": 8, "f32": 4, "f16": 2, "bf16": 2}


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def _prod(xs):
    p = 1
    for x in xs:
        p *= int(x)
    return p


# ------------------------------------------------------------ partition --
def plan(workload: str, rank: int, world: int, scaling: str | None = None) -> dict:
    """This rank's share of the workload: block-row slab [r0, r1) of axis 0
    of the global array (same rule as paper_2406_11209_b200.distributed)."""
    w = WORKLOADS[workload]
    scaling = scaling or w["scaling"]
    shape, block = tuple(w["shape"]), tuple(w["block"])
    if scaling == "weak":
        global_shape = (shape[0] * world,) + shape[1:]
    else:
        global_shape = shape
    g0 = -(-global_shape[0] // block[0])
    b0, b1 = (g0 * rank) // world, (g0 * (rank + 1)) // world
    r0, r1 = b0 * block[0], min(b1 * block[0], global_shape[0])
    local = (r1 - r0,) + global_shape[1:]
    row = _prod(global_shape[1:])
    return {"workload": workload, "scaling": scaling, "rank": rank, "world": world,
            "global_shape": list(global_shape), "local_shape": list(local), "rows": [r0, r1],
            "offset": r0 * row, "local_elems": _prod(local), "global_elems": _prod(global_shape)}


def input_fields(workload: str) -> int:
    return 2 if WORKLOADS[workload]["step"] == "pair" else 1


def config_dict(workload: str, world: int, scaling: str | None = None) -> dict:
    """The `config` object -- identical for both arms (ours / reference)."""
    w = WORKLOADS[workload]
    p = plan(workload, 0, world, scaling)
    kept = _prod(w["block"]) if w["lowpass"] is None else None
    if kept is None:
        import itertools
        kept = sum(1 for idx in itertools.product(*[range(b) for b in w["block"]])
                   if sum(idx) <= w["lowpass"])
    in_bytes = p["local_elems"] * ITEMSIZE[w["fk"]]
    return {
        "workload": w["desc"],
        "name": workload,
        "global_shape": p["global_shape"],
        "per_gpu_shape": p["local_shape"],
        "block": list(w["block"]),
        "float_kind": w["fk"],
        "index_kind": w["ik"],
        "kept": kept,
        "fields": input_fields(workload),
        "scaling": p["scaling"],
        "parallelism": f"block-row shards x{world}; one all_gather_into_tensor of 16-double "
                       f"records per reduction",
        "l2_flush": f"not needed: inputs are {in_bytes / 2**20:.0f} MiB per GPU per field > "
                    f"126 MB L2",
    }


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


# ------------------------------------------------------------- launcher --
def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_cmd(argv, nproc: int, port: int) -> list:
    """torchrun command re-running this script with one process per GPU."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", f"--master-port={port}",
            os.path.abspath(__file__), *argv]


class Group:
    """Process-group plumbing shared by the GPU and dry-run paths."""

    def __init__(self, world: int, rank: int, local: int, backend: str, device=None):
        import torch.distributed as dist

        self.world, self.rank, self.local = world, rank, local
        self.dist = dist
        self.device = device
        if world > 1 and not dist.is_initialized():
            kw = {"device_id": device} if backend == "nccl" else {}
            dist.init_process_group(backend, **kw)

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, v: float) -> float:
        if self.world == 1:
            return v
        import torch

        dev = self.device if self.dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def gather_into(self, rec):
        """[world * numel] tensor of every rank's `rec` (one collective)."""
        if self.world == 1:
            return rec
        import torch

        if self.dist.get_backend() != "nccl" and rec.is_cuda:  # --share-gpu check runs (gloo)
            return self.gather_into(rec.cpu()).to(rec.device)
        out = torch.empty(self.world * rec.numel(), dtype=rec.dtype, device=rec.device)
        self.dist.all_gather_into_tensor(out, rec.reshape(-1))
        return out

    def gather_objects(self, obj):
        if self.world == 1:
            return [obj]
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out

    def close(self):
        if self.world > 1 and self.dist.is_initialized():
            self.dist.barrier()
            self.dist.destroy_process_group()


def run_dry(args):
    """Rank orchestration without kernels (CPU, gloo): every rank's plan and
    a max-over-ranks timing round trip; rank 0 prints one JSON line."""
    import torch

    world, rank = env_int("WORLD_SIZE", 1), env_int("RANK", 0)
    g = Group(world, rank, env_int("LOCAL_RANK", 0), "gloo", torch.device("cpu"))
    p = plan(args.workload, rank, world, args.scaling)
    plans = g.gather_objects(p)
    rec = torch.full((16,), float(rank + 1), dtype=torch.float64)
    gathered = g.gather_into(rec).reshape(world, -1)[:, 0].tolist()
    t = g.max(float(rank + 1))
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "max_over_ranks": t,
                          "records": gathered, "plans": plans,
                          "config": config_dict(args.workload, world, args.scaling)}))
    g.close()


# --------------------------------------------------------------------- ours --
def run_ours(args):
    import numpy as np
    import torch

    import paper_2406_11209_b200 as bz
    from paper_2406_11209_b200 import _native
    from paper_2406_11209_b200 import distributed as bd
    from paper_2406_11209_b200.ops import Record, merge_records, moments_record

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    # --share-gpu (check runs only): every rank on cuda:0 over gloo, so the
    # multi-rank path can be exercised on a one-GPU box; timings meaningless
    local = 0 if args.share_gpu else env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    g = Group(world, rank, local, "gloo" if args.share_gpu else "nccl", dev)

    w = WORKLOADS[args.workload]
    p = plan(args.workload, rank, world, args.scaling)
    shape, gshape = tuple(p["local_shape"]), tuple(p["global_shape"])
    kind = bz.FloatKind(w["fk"])
    mask = None
    if w["lowpass"] is not None:
        mask = bz.PruningMask(w["block"], np.indices(w["block"]).sum(axis=0) <= w["lowpass"])
    s = bz.CodecSettings(w["block"], kind, bz.IndexKind(w["ik"]), bz.TransformFamily.DCT, mask)
    n_local = p["local_elems"]
    fields = input_fields(args.workload)
    in_bytes_local = n_local * kind.itemsize * fields
    in_bytes_total = p["global_elems"] * kind.itemsize * fields
    B = int(np.prod(s.grid_for(shape)))
    K = s.mask.kept_count
    comp_bytes = B * (K * s.index_kind.itemsize + kind.itemsize)
    stream = torch.cuda.current_stream(dev)

    def field(seed, dist_=0):
        t = torch.empty(shape, dtype=kind.torch_dtype, device=dev)
        _native.call("bz_fill_random", t.data_ptr(), kind.code, n_local, p["offset"], seed, dist_,
                     _native.stream_handle(dev))
        return bz.DenseArray.wrap(t, kind)

    # synthetic inputs: counter-based, partition invariant (global flat offset)
    xa = field(2)
    ya = field(3) if w["step"] in ("chain", "pair", "sweep") else None
    cy = bz.compress(ya, s) if w["step"] in ("chain", "sweep") else None

    def shard(c):
        return bd.ShardedCompressedArray(c, gshape) if world > 1 else c

    kind_step = w["step"]
    outs = []

    # ---- one device-resident step: no host synchronisation inside
    def step():
        if kind_step == "codec":
            ca = bz.compress(xa, s)
            rec = g.gather_into(moments_record(ca, dc_only=2))  # "sums": what l2_norm uses
            out = bz.decompress(ca)
            outs.append(rec)
            return out
        if kind_step == "chain":
            cx = bz.compress(xa, s)
            m = bz.mul_scalar(bz.add(cx, cy), 0.5)
            outs.append(g.gather_into(moments_record(m)))  # mean + variance record
            return m
        if kind_step == "pair":
            cx, cy2 = bz.compress(xa, s), bz.compress(ya, s)
            outs.append(g.gather_into(moments_record(cx, cy2)))  # cov / cosine / ssim record
            return cx
        # sweep
        cx = bz.compress(xa, s)
        sq = torch.empty(1, dtype=torch.float64, device=dev)
        if not bz.ops._subtract_l2_sq(cx, cy, sq):
            raise RuntimeError("fused subtract+l2 does not serve this configuration")
        outs.append(g.gather_into(sq))
        return bz.decompress(cx)

    def timed(fn, reps):
        g.barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        g.barrier()
        return g.max(e0.elapsed_time(e1) / reps)

    with ClockSampler(dev) as clocks:
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize(dev)
        outs.clear()
        launches0 = _native.query("bz_launch_count")
        clocks.mark(True)
        ms_step = timed(step, args.steps)
        clocks.mark(False)
        launches = _native.query("bz_launch_count") - launches0
    value = in_bytes_total / (ms_step * 1e-3) / 1e9

    # ---- results of the timed steps (host epilogue, after the timed region)
    r = s.index_kind.radius

    def merged(t):
        h = t.cpu().numpy().reshape(world, -1)
        return merge_records([Record.from_array(h[i]) for i in range(world)])

    check = {}
    if kind_step == "codec":
        vals = []
        for t in outs:
            rr = merged(t)
            vals.append(math.sqrt(max(rr.s_aa, 0.0)) / r)
        check = {"l2_norm": vals[-1], "identical_over_steps": len(set(vals)) == 1}
    elif kind_step == "chain":
        rr = merged(outs[-1])
        c = s.block_mean_scale
        nb_total = int(np.prod(s.grid_for(gshape)))
        check = {"mean": (rr.mean_a / r) / c,
                 "variance": (rr.m_aa + rr.s_aa) / (r * r) / (nb_total * s.block_size)}
    elif kind_step == "pair":
        rr = merged(outs[-1])
        nb_total = int(np.prod(s.grid_for(gshape)))
        cov = (rr.m_ab + rr.s_ab) / (r * r) / (nb_total * s.block_size)
        na = math.sqrt(rr.s_aa + rr.m_aa + rr.n * rr.mean_a ** 2)
        nb = math.sqrt(rr.s_bb + rr.m_bb + rr.n * rr.mean_b ** 2)
        check = {"covariance": cov,
                 "cosine": (rr.s_ab + rr.m_ab + rr.n * rr.mean_a * rr.mean_b) / (na * nb)}
    else:
        h = outs[-1].cpu().numpy().reshape(-1)
        check = {"l2_diff": math.sqrt(max(float(sum(h)), 0.0)) / r}

    # ---- per-op breakdown (same kernels, timed one by one)
    ca = bz.compress(xa, s)
    reps = max(args.steps, 5)
    ops = {}
    peak, peak_src = load_peak()
    n_bytes_field = n_local * kind.itemsize

    def op(name, fn, alg_bytes, in_bytes):
        for _ in range(3):
            fn()
        ms = timed(fn, reps)
        ops[name] = {"ms": round(ms, 5), "gbs_uncompressed": round(in_bytes / ms / 1e6, 1),
                     "gbs_algorithmic": round(alg_bytes / ms / 1e6, 1),
                     "roofline_frac": round(alg_bytes / ms / 1e6 / peak, 4),
                     "alg_bytes": alg_bytes}

    op("compress", lambda: bz.compress(xa, s), n_bytes_field + comp_bytes, n_bytes_field)
    if kind_step in ("codec", "sweep"):
        op("decompress", lambda: bz.decompress(ca), comp_bytes + n_local * 8, n_bytes_field)
    if kind_step == "codec":
        op("l2_norm", lambda: g.gather_into(moments_record(ca, dc_only=2)), comp_bytes,
           n_bytes_field)
        cb = bz.compress(bz.DenseArray.wrap(torch.flip(xa.values, dims=[0]).contiguous(), kind), s)
        op("dot", lambda: g.gather_into(moments_record(ca, cb, dc_only=2)), 2 * comp_bytes,
           2 * n_bytes_field)
    if kind_step == "chain":
        op("add", lambda: bz.add(ca, cy), 3 * comp_bytes, 2 * n_bytes_field)
        op("mul_scalar", lambda: bz.mul_scalar(ca, 0.5), B * kind.itemsize * 2, n_bytes_field)
        op("mean_variance", lambda: g.gather_into(moments_record(ca)), comp_bytes, n_bytes_field)
        op("mean", lambda: g.gather_into(moments_record(ca, dc_only=1)),
           B * (s.index_kind.itemsize + kind.itemsize), n_bytes_field)
    if kind_step == "pair":
        cb = bz.compress(ya, s)
        op("cov_cos_ssim", lambda: g.gather_into(moments_record(ca, cb)), 2 * comp_bytes,
           2 * n_bytes_field)
    if kind_step == "sweep":
        sq = torch.empty(1, dtype=torch.float64, device=dev)
        op("subtract_l2", lambda: bz.ops._subtract_l2_sq(ca, cy, sq), 2 * comp_bytes,
           2 * n_bytes_field)
    dominant = max(ops, key=lambda k: ops[k]["ms"])
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

    # ---- end to end through the public API from pinned host memory
    e2e = run_e2e(args, bz, bd, torch, dev, stream, g, s, kind, shape, gshape, xa, ya, cy,
                  kind_step, n_local, in_bytes_local, in_bytes_total, world)

    result = None
    if rank == 0:
        cpu = parity = None
        if world == 1 and not args.no_cpu_baseline:
            cpu, parity = cpu_leg(args.workload, dev)
        result = {
            "metric": METRIC,
            "value": round(value, 3),
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_step, 5),
            "higher_is_better": True,
            "scaling": p["scaling"],
            "vs_baseline": None,
            "dtype": w["fk"],
            "data": "synthetic: counter-based N(0,1), partition-invariant (bz_fill_random)",
            "config": config_dict(args.workload, world, args.scaling),  # == the reference arm's
            "fast_path": bz.is_fast_path(s, shape),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "parity": parity,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
            "ops": ops,
            "check": check,
        }
        print(json.dumps(result))
    g.close()
    return result


def run_e2e(args, bz, bd, torch, dev, stream, g, s, kind, shape, gshape, xa, ya, cy, kind_step,
            n_local, in_bytes_local, in_bytes_total, world):
    """The step through the public API from pinned host memory.  For the
    codec step two CUDA streams alternate, so step i's D2H copy of the
    decompressed array overlaps step i+1's H2D copy (PCIe is full duplex);
    every step still pays its own H2D, D2H and scalar read-backs."""

    def shard(c):
        return bd.ShardedCompressedArray(c, gshape) if world > 1 else c

    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    nbuf = 2 if kind_step == "codec" else 1  # only the codec step alternates streams
    host_x = [torch.empty(shape, dtype=kind.torch_dtype, pin_memory=True) for _ in range(nbuf)]
    for h in host_x:
        h.copy_(xa.values.cpu())
    host_y = None
    if kind_step == "pair":
        host_y = torch.empty(shape, dtype=kind.torch_dtype, pin_memory=True)
        host_y.copy_(ya.values.cpu())
    decomp = kind_step in ("codec", "sweep")
    host_out = [torch.empty(shape, dtype=torch.float64, pin_memory=True) for _ in range(nbuf)] \
        if decomp else None
    results = []
    it = [0]
    d2h_scalars = {"codec": 1, "chain": 2, "pair": 3, "sweep": 1}[kind_step]

    def e2e_step():
        i = it[0] % nbuf
        it[0] += 1
        st = streams[i] if kind_step == "codec" else stream
        with torch.cuda.stream(st):
            a = bz.DenseArray(shape, kind, host_x[i])       # H2D copy (async, pinned)
            c = shard(bz.compress(a, s))
            if kind_step == "codec":
                results.append(bz.l2_norm(c))
            elif kind_step == "chain":
                m = bz.mul_scalar(bz.add(c, shard(cy)), 0.5)
                results.append((bz.mean(m), bz.variance(m)))
            elif kind_step == "pair":
                c2 = shard(bz.compress(bz.DenseArray(shape, kind, host_y), s))
                results.append((bz.covariance(c, c2), bz.cosine_similarity(c, c2),
                                bz.ssim(c, c2)))
            else:
                results.append(bz.subtract_l2(c, shard(cy)))
            if decomp:
                out = bz.decompress(c)
                host_out[i].copy_(out.values, non_blocking=True)  # D2H copy of the result

    def e2e_timed(reps):
        g.barrier()
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
        g.barrier()
        return g.max(e0.elapsed_time(e1) / reps)

    e2e_steps = max(8, args.steps // 2)
    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize(dev)
    ms_e2e = e2e_timed(e2e_steps)
    paths = {
        "codec": "DenseArray(pinned host) -> compress -> l2_norm -> decompress -> host copy; two "
                 "streams alternate so D2H of step i overlaps H2D of step i+1",
        "chain": "DenseArray(pinned host) -> compress -> add -> mul_scalar -> mean, variance",
        "pair": "two DenseArrays(pinned host) -> compress x2 -> covariance, cosine_similarity, "
                "ssim",
        "sweep": "DenseArray(pinned host) -> compress -> subtract_l2 (fused) -> decompress -> "
                 "host copy",
    }
    return {
        "value": round(in_bytes_total / (ms_e2e * 1e-3) / 1e9, 3),
        "unit": "GB/s",
        "h2d_bytes_per_step": in_bytes_local,
        "d2h_bytes_per_step": (n_local * 8 if decomp else 0) + 8 * d2h_scalars,
        "ms_per_step": round(ms_e2e, 4),
        "steps": e2e_steps,
        "path": paths[kind_step],
    }


# ---------------------------------------------------------------- CPU side --
def _slab_rows(workload: str) -> int:
    """Rows of the bounded CPU sample: about 8M elements, whole block rows."""
    w = WORKLOADS[workload]
    shape, block = w["shape"], w["block"]
    row = _prod(shape[1:])
    rows = max(block[0], (8 * 2**20 // row) // block[0] * block[0])
    return min(rows, shape[0])


class CpuImpl:
    """The reference package ``bzc`` (baseline/_ref, kind "reference") or,
    when it is not installed, the numpy oracle port (kind "port")."""

    def __init__(self, workload: str, prefer_reference: bool = True):
        import numpy as np

        w = WORKLOADS[workload]
        self.w = w
        self.bits = None if w["lowpass"] is None else \
            (np.indices(w["block"]).sum(axis=0) <= w["lowpass"])
        ref = os.path.join(ROOT, "baseline", "_ref")
        self.kind = "port"
        if prefer_reference and os.path.isdir(os.path.join(ref, "bzc")):
            if ref not in sys.path:
                sys.path.insert(0, ref)
            try:
                import bzc

                self.bzc = bzc
                self.kind = "reference"
                self.settings = bzc.CodecSettings(
                    w["block"], bzc.FloatKind(w["fk"]), bzc.IndexKind(w["ik"]),
                    bzc.TransformFamily.DCT,
                    None if self.bits is None else bzc.PruningMask(w["block"], self.bits))
            except Exception:
                self.kind = "port"
        if self.kind == "port":
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            import bzc_oracle as o

            self.o = o
            self.settings = o.Settings(w["block"], w["fk"], w["ik"], "dct", self.bits)

    def compress(self, x):
        if self.kind == "reference":
            b = self.bzc
            return b.compress(b.DenseArray(x.shape, b.FloatKind(self.w["fk"]), x), self.settings)
        return self.o.compress(x, self.settings)

    def decompress(self, c):
        if self.kind == "reference":
            return self.bzc.decompress(c).values
        return self.o.decompress(c)

    def __getattr__(self, name):  # l2_norm, add, mul_scalar, mean, variance, ...
        mod = self.__dict__.get("bzc") if self.__dict__.get("kind") == "reference" \
            else self.__dict__.get("o")
        return getattr(mod, name)

    def step(self, x, y=None, cy=None):
        """One CPU step of the workload; returns its scalar results."""
        st = self.w["step"]
        if st == "codec":
            c = self.compress(x)
            v = self.l2_norm(c)
            self.decompress(c)
            return (v,)
        if st == "chain":
            m = self.mul_scalar(self.add(self.compress(x), cy), 0.5)
            return (self.mean(m), self.variance(m))
        if st == "pair":
            a, b = self.compress(x), self.compress(y)
            return (self.covariance(a, b), self.cosine_similarity(a, b), self.ssim(a, b))
        c = self.compress(x)
        v = self.l2_norm(self.add(c, self.negate(cy)))
        self.decompress(c)
        return (v,)


def _cpu_inputs(workload, rows, seed):
    import numpy as np

    w = WORKLOADS[workload]
    rng = np.random.default_rng(seed)
    shp = (rows,) + tuple(w["shape"][1:])
    dt = np.float32 if w["fk"] == "f32" else np.float64
    x = rng.normal(size=shp).astype(dt).astype(np.float64)
    y = (0.5 * x + 0.5 * rng.normal(size=shp)).astype(dt).astype(np.float64)
    return x, y


def cpu_leg(workload, dev, min_seconds=10.0, max_reps=10):
    """cpu_baseline (the reference on ONE core, bounded slab) and parity of the
    GPU path against the reference's outputs on the same slab."""
    try:
        from threadpoolctl import threadpool_limits
    except Exception:  # pragma: no cover
        threadpool_limits = None
    rows = _slab_rows(workload)
    impl = CpuImpl(workload)
    x, y = _cpu_inputs(workload, rows, 2)
    w = WORKLOADS[workload]
    cy = impl.compress(y) if w["step"] in ("chain", "sweep") else None
    nbytes = x.size * ITEMSIZE[w["fk"]] * input_fields(workload)
    ctx = threadpool_limits(limits=1) if threadpool_limits else None
    if ctx:
        ctx.__enter__()
    try:
        want = impl.step(x, y, cy)
        times = []
        t_all = time.perf_counter()
        while len(times) < max_reps and (time.perf_counter() - t_all) < min_seconds:
            t0 = time.perf_counter()
            impl.step(x, y, cy)
            times.append(time.perf_counter() - t0)
    finally:
        if ctx:
            ctx.__exit__(None, None, None)
    t = statistics.median(times)
    cpu = {
        "value": round(nbytes / t / 1e9, 4),
        "unit": "GB/s",
        "cores": 1,
        "kind": impl.kind,
        "sample": f"{rows}x{'x'.join(map(str, w['shape'][1:]))} slab ({x.size} elements per "
                  f"field); the workload's step; median of {len(times)} reps ({t:.3f} s each); "
                  f"{'bzc from baseline/_ref' if impl.kind == 'reference' else 'numpy oracle port'}"
                  f", BLAS 1 thread",
    }
    try:
        parity = gpu_parity(workload, impl, x, y, cy, want, dev)
    except Exception as e:  # report, never hide
        parity = {"error": f"{type(e).__name__}: {e}"}
    return cpu, parity


def gpu_parity(workload, impl, x, y, cy, want, dev):
    """The GPU path on the CPU sample vs the reference's outputs: indices
    bit-exact except at rounding ties (reported), maxima bit-exact,
    decompression and operator results within the stated tolerances."""
    import numpy as np
    import torch

    import paper_2406_11209_b200 as bz

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import bzc_oracle as o  # the checker's tie detector

    w = WORKLOADS[workload]
    kind = bz.FloatKind(w["fk"])
    mask = None if impl.bits is None else bz.PruningMask(w["block"], impl.bits)
    s = bz.CodecSettings(w["block"], kind, bz.IndexKind(w["ik"]), bz.TransformFamily.DCT, mask)
    ga = bz.compress(bz.DenseArray(x.shape, kind, torch.from_numpy(x).to(dev)), s)
    ref = impl.compress(x)
    ref_idx = np.asarray(ref.indices)
    ref_max = np.asarray(ref.maxima_f64() if hasattr(ref, "maxima_f64") else ref.maxima,
                         dtype=np.float64)
    got_idx = ga.indices.cpu().numpy()
    got_max = ga.maxima_f64().cpu().numpy()
    os_ = o.Settings(w["block"], w["fk"], w["ik"], "dct", impl.bits)
    coeffs = o.coefficients(x, os_)
    ties = o.prune_and_flatten(o.tie_mask(coeffs, ref_max, len(w["block"]), w["ik"]),
                               os_.mask_bits)
    diff = got_idx != ref_idx
    out = bz.decompress(ga).values.cpu().numpy()
    ref_out = np.asarray(impl.decompress(ref))
    scale = float(np.max(np.abs(ref_out))) or 1.0
    res = {
        "sample_elements": int(x.size),
        "reference": impl.kind,
        "indices": int(ref_idx.size),
        "index_mismatches": int(diff.sum()),
        "index_mismatches_off_tie": int((diff & ~ties).sum()),
        "tie_fraction": float(ties.sum()) / max(1, ties.size),
        "maxima_bit_exact": bool(np.array_equal(got_max.view(np.int64), ref_max.view(np.int64))),
        "decompress_max_rel_err": float(np.max(np.abs(out - ref_out)) / scale),
        "decompress_tolerance": 1e-13,
        "op_tolerance": 1e-9,
    }
    st = w["step"]
    if st == "codec":
        got = (bz.l2_norm(ga),)
    else:
        gy = bz.compress(bz.DenseArray(y.shape, kind, torch.from_numpy(y).to(dev)), s)
        if st == "chain":
            m = bz.mul_scalar(bz.add(ga, gy), 0.5)
            got = (bz.mean(m), bz.variance(m))
        elif st == "pair":
            got = (bz.covariance(ga, gy), bz.cosine_similarity(ga, gy), bz.ssim(ga, gy))
        else:
            got = (bz.subtract_l2(ga, gy),)
    res["op_values"] = [float(v) for v in got]
    res["op_max_rel_err"] = max(abs(a - b) / max(abs(b), 1e-300) for a, b in zip(got, want))
    return res


_W = {}


def _ref_init(workload, rows, seed):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    impl = CpuImpl(workload)
    x, y = _cpu_inputs(workload, rows, seed)
    _W.update(impl=impl, x=x, y=y,
              cy=impl.compress(y) if WORKLOADS[workload]["step"] in ("chain", "sweep") else None)


def _ref_task(_):
    return _W["impl"].step(_W["x"], _W["y"], _W["cy"])


def run_reference(args):
    """The reference package on every host core: one process per core, each
    running the workload's step on its own block-row slab."""
    rank = env_int("RANK", 0)
    if rank != 0:
        return None
    import multiprocessing as mp

    w = WORKLOADS[args.workload]
    procs = max(1, os.cpu_count() or 1)
    rows_per = max(w["block"][0], _slab_rows(args.workload) // 4 // w["block"][0] * w["block"][0])
    ctx = mp.get_context("spawn")
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    pools = [ctx.Pool(1, initializer=_ref_init, initargs=(args.workload, rows_per, 100 + i))
             for i in range(procs)]
    kind = CpuImpl(args.workload).kind
    try:
        def one_step():
            res = [p.apply_async(_ref_task, (0,)) for p in pools]
            return [r.get() for r in res]

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
    elem = rows_per * procs * _prod(w["shape"][1:])
    nbytes = elem * ITEMSIZE[w["fk"]] * input_fields(args.workload)
    t = statistics.mean(times)
    value = nbytes / t / 1e9
    sample = (f"{rows_per * procs}x{'x'.join(map(str, w['shape'][1:]))} per step ({rows_per} "
              f"rows per process x {procs} processes); the workload's step; "
              f"{'bzc from baseline/_ref' if kind == 'reference' else 'numpy oracle port'}")
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
        "scaling": plan(args.workload, 0, args.gpus, args.scaling)["scaling"],
        "vs_baseline": None,
        "dtype": w["fk"],
        "data": "synthetic: numpy N(0,1)",
        "config": config_dict(args.workload, args.gpus, args.scaling),
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": procs, "kind": kind,
                         "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))
    return out


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", choices=sorted(WORKLOADS), default="c2")
    p.add_argument("--scaling", choices=["weak", "strong"], default=None)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--dry-run", action="store_true",
                   help="rank orchestration only (CPU/gloo): plans + one max-over-ranks")
    p.add_argument("--share-gpu", action="store_true",
                   help="check runs: all ranks on cuda:0 over gloo (not a measurement)")
    args = p.parse_args(argv)
    args.warmup = max(3, args.warmup)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        # one process per GPU: re-run this script under torchrun
        rc = subprocess.call(relaunch_cmd(argv, args.gpus, _free_port()))
        sys.exit(rc)
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
