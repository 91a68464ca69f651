"""World-size-2 gloo test of the multi-GPU host logic (CPU): contiguous group
shards, the per-group size gather and max-over-ranks timing used by bench.py."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2008_06972_b200 import dist as pdist

    lo, hi = pdist.shard_range(10, rank, world)
    local = torch.arange(lo, hi, dtype=torch.int64) * 100
    if local.numel() < 5:  # equal-length gather
        local = torch.cat([local, torch.full((5 - local.numel(),), -1, dtype=torch.int64)])
    sizes = pdist.gather_sizes(local)
    t = pdist.max_over_ranks(1.5 + rank, "cpu")
    s = pdist.sum_over_ranks(hi - lo, "cpu")
    q.put((rank, (lo, hi), sizes.tolist(), t, s))
    dist.destroy_process_group()


def test_shard_range_covers_all_groups():
    from paper_2008_06972_b200.dist import shard_range

    for n in (0, 1, 7, 1024, 1025):
        for world in (1, 2, 4, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def test_gloo_world2_gather_and_max():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, sh0, sz0, t0, s0), (r1, sh1, sz1, t1, s1) = res
    assert sh0 == (0, 5) and sh1 == (5, 10)
    assert sz0 == sz1 == [i * 100 for i in range(10)]
    assert t0 == t1 == 2.5
    assert s0 == s1 == 10


def _ragged_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2008_06972_b200 import dist as pdist

    out = {}
    for n_total in (1025, 1024, 3, 1):
        lo, hi = pdist.shard_range(n_total, rank, world)
        local = torch.arange(lo, hi, dtype=torch.int64) * 7 + 3  # "blob size" of group g
        out[n_total] = pdist.gather_ragged(local, n_total, world).tolist()
    q.put((rank, out))
    dist.destroy_process_group()


def test_gloo_world2_strong_scaling_ragged_gather():
    """bench.py's strong-scaling mode: one fixed batch split by contiguous
    group shards (also odd totals, and more ranks than groups), per-group
    sizes gathered back in group order with the padding stripped."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ragged_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for n_total in (1025, 1024, 3, 1):
        want = [g * 7 + 3 for g in range(n_total)]
        assert res[0][n_total] == res[1][n_total] == want


def test_numa_helpers_tolerate_unknown_topology():
    from paper_2008_06972_b200 import dist as pdist

    assert pdist._cpulist("0-3,8,10-11") == [0, 1, 2, 3, 8, 10, 11]
    info = pdist.bind_to_gpu_numa(0)  # no GPU here: a no-op report
    assert "numa_node" in info
