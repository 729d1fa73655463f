"""Multi-process (world_size 2, gloo, CPU) coverage of the N > 1 path:
batch partition across ranks, each rank's host-side geometry of its own
shard (smol_debug_geometry, no GPU), the max-over-ranks timing reduction,
and bench.py's torchrun launch of the reference arm over gloo."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2007_13005_b200 import shard


def test_partition_properties():
    for n in (0, 1, 3, 7, 256, 1000):
        for world in (1, 2, 3, 4, 8):
            w = [1 + (i * 37) % 5 for i in range(n)]
            parts = shard.partition(w, world)
            assert len(parts) == world
            assert parts[0][0] == 0 and parts[-1][1] == n
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c and a <= b
            if n >= world * 4:
                sums = [sum(w[a:b]) for a, b in parts]
                assert max(sums) - min(sums) <= 2 * max(w)


def test_partition_heterogeneous_balance():
    w = [2688] * 100 + [48720] * 10          # c2-sized and c5-sized images
    parts = shard.partition(w, 4)
    sums = [sum(w[a:b]) for a, b in parts]
    assert max(sums) <= 1.3 * (sum(w) / 4) + max(w)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = [100 + (i % 7) for i in range(64)]
        parts = shard.partition(w, world)
        lo, hi = parts[rank]
        # every rank derives the same partition; its share is disjoint
        mine = list(range(lo, hi))
        got = shard.max_over_ranks(10.0 + rank)
        import torch
        t = torch.tensor([len(mine)])
        dist.all_reduce(t)
        # per-rank geometry of its own shard of a heterogeneous c2-style
        # batch, gathered over gloo: every image exactly once, and each
        # image's ROI block count equals the single-process value
        import paper_2007_13005_b200 as smol
        import synth
        ps = smol.params_from_config(synth.CONFIGS["c2"])
        sizes = [(500, 375), (375, 500), (640, 480), (97, 61), (1920, 1080), (161, 161)] * 5
        ims = [type("I", (), {"width": a, "height": b})() for a, b in sizes]
        wts = shard.roi_weights(ps, ims)
        a, b = shard.partition(wts, world)[rank]
        mine_geo = [(i, smol.geometry(ps, *sizes[i])["roi_blocks"]) for i in range(a, b)]
        gathered = [None] * world
        dist.all_gather_object(gathered, mine_geo)
        q.put((rank, lo, hi, got, int(t.item()), gathered, wts))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_shards_and_max_time():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1] == 0 and res[0][2] == res[1][1] and res[1][2] == 64
    assert all(r[3] == 11.0 for r in res)          # max over ranks
    assert all(r[4] == 64 for r in res)            # every image exactly once
    gathered, wts = res[0][5], res[0][6]
    flat = [x for part in gathered for x in part]
    assert [i for i, _ in flat] == list(range(len(wts)))        # disjoint, contiguous, complete
    assert [b for _, b in flat] == wts                           # per-rank geometry == single process
    sums = [sum(b for _, b in part) for part in gathered]
    assert max(sums) <= sum(wts) / 2 + max(wts)                  # ROI-balanced


def test_bench_reference_arm_torchrun_gloo(tmp_path):
    """bench.py --impl reference under torchrun with 2 ranks (gloo, CPU):
    rank 0 prints one JSON line, rank 1 exits 0 without work."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(root, "bench.py"), "--impl", "reference", "--config", "c1", "--gpus", "2",
           "--steps", "2", "--warmup", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"] == {"workload": d["config"]["workload"]}
