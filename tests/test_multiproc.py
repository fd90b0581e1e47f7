"""World-size-2 (gloo, CPU) coverage of the multi-GPU host logic: session
sharding is a partition with no data-path exchange, and bench.py's
max-over-ranks timing reduction."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_08699_b200.sessions import (config5_scene_size, config5_sessions, scenes_for,
                                            shard)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = shard(config5_sessions(64), rank, world)
        ids = [None] * world
        dist.all_gather_object(ids, [s.index for s in mine])
        # bench.py: per-rank elapsed, MAX over ranks
        t = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            out.put((ids, float(t.item()), scenes_for(mine)))
    finally:
        dist.destroy_process_group()


def test_session_partition_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ids, tmax, scenes0 = q.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    flat = sorted(ids[0] + ids[1])
    assert flat == list(range(64))
    assert not set(ids[0]) & set(ids[1])
    assert tmax == 2.0
    # rank 0 of 2 serves even sessions -> even scene sizes only
    assert scenes0 == [0, 2, 4, 6, 8, 10, 12]


def test_config5_sizes():
    sizes = [config5_scene_size(k) for k in range(14)]
    assert sizes[0] == 250_000 and sizes[-1] == 6_000_000
    assert all(a < b for a, b in zip(sizes, sizes[1:]))


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_shard_is_partition(world):
    sess = config5_sessions(64)
    parts = [shard(sess, r, world) for r in range(world)]
    assert sorted(s.index for p in parts for s in p) == list(range(64))
    assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1
    with pytest.raises(ValueError):
        shard(sess, world, world)


def _bench_dry(*extra):
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--dry-run", "--steps", "8",
                        "--warmup", "3", *extra], capture_output=True, text=True, timeout=300,
                       cwd=root, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints one JSON line
    return json.loads(lines[0])


def test_bench_gpus2_launches_two_ranks():
    """`bench.py --gpus 2` without a torchrun environment re-launches itself
    with two ranks (torch.distributed.run, 127.0.0.1); each rank owns its own
    session trace and rank 0 reports n_gpus = 2 after the max-over-ranks."""
    line = _bench_dry("--gpus", "2")
    assert line["n_gpus"] == 2 and line["dry_run"] is True
    assert line["sessions_by_rank"] == [[0], [1]]


def test_bench_config5w_weak_sharding_two_ranks():
    """config 5w: 8 sessions per GPU, session i -> GPU i mod N."""
    line = _bench_dry("--gpus", "2", "--workload", "config5w")
    assert line["n_gpus"] == 2 and line["sessions"] == 16
    assert line["sessions_by_rank"] == [list(range(0, 16, 2)), list(range(1, 16, 2))]


def test_bench_single_process_dry_run():
    line = _bench_dry()
    assert line["n_gpus"] == 1 and line["sessions_by_rank"] == [[0]]
