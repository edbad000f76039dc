"""bench.py's multi-GPU orchestration on CPU (gloo, world size 2).

The driver runs ``bench.py --gpus N``; without a torchrun environment the
script must re-launch itself with one process per GPU.  ``--dry-run`` runs
exactly that launch + process-group + partition + max-over-ranks + record
all-gather path with the gloo backend and no kernels.
"""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


@pytest.mark.parametrize("workload", sorted(bench.WORKLOADS))
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_plan_partitions_like_the_library(workload, world):
    from paper_2406_11209_b200 import distributed as bd

    plans = [bench.plan(workload, r, world) for r in range(world)]
    g = plans[0]["global_shape"]
    block = bench.WORKLOADS[workload]["block"]
    assert plans[0]["rows"][0] == 0 and plans[-1]["rows"][1] == g[0]
    for r, p in enumerate(plans):
        assert tuple(p["rows"]) == bd.shard_slab(g, block, r, world)
        assert p["local_shape"] == [p["rows"][1] - p["rows"][0]] + g[1:]
    assert sum(p["local_elems"] for p in plans) == plans[0]["global_elems"]
    if plans[0]["scaling"] == "strong":
        assert g == list(bench.WORKLOADS[workload]["shape"])
    else:
        assert g[0] == bench.WORKLOADS[workload]["shape"][0] * world


def test_config_identical_for_both_arms():
    for wl in bench.WORKLOADS:
        for world in (1, 8):
            assert bench.config_dict(wl, world) == bench.config_dict(wl, world)
    c = bench.config_dict("c5", 1)
    assert c["kept"] == 66 and c["scaling"] == "strong"


def test_self_launch_two_ranks_dry_run():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--dry-run", "--workload", "c3"],
                         capture_output=True, text=True, timeout=240, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["dry_run"]
    assert rec["max_over_ranks"] == 2.0          # max of (1, 2)
    assert rec["records"] == [1.0, 2.0]          # one all_gather_into_tensor, rank order
    assert [p["rank"] for p in rec["plans"]] == [0, 1]
    assert rec["plans"][0]["rows"] == [0, 512] and rec["plans"][1]["rows"] == [512, 1024]
    assert rec["config"]["scaling"] == "strong"


def test_relaunch_command_uses_loopback():
    cmd = bench.relaunch_cmd(["--gpus", "4"], 4, 12345)
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-2:] == ["--gpus", "4"]
