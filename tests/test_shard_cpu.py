"""Multi-process sharding logic on CPU (gloo, world_size 2): shard ranges,
global output placement via the all-gathered byte totals.  The per-GPU step is
replaced by a CPU stand-in built on the oracle (test infrastructure only)."""

import os
import socket

import numpy as np
import pytest

from paper_2305_09493_b200.shard import local_batch, shard_ranges


def test_shard_ranges_cover_and_balance():
    rng = np.random.default_rng(3)
    lengths = rng.integers(20, 6000, size=1001) // 4 * 4
    for world in (1, 2, 3, 8):
        r = shard_ranges(lengths, world)
        assert r[0][0] == 0 and r[-1][1] == len(lengths)
        assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
        sizes = [int(lengths[a:b].sum()) for a, b in r]
        assert max(sizes) - min(sizes) <= 2 * int(lengths.max())
    assert shard_ranges([], 4) == [(0, 0)] * 4
    assert [b - a for a, b in shard_ranges([8, 8], 4)] == [0, 1, 0, 1] or \
        sum(b - a for a, b in shard_ranges([8, 8], 4)) == 2


def test_local_batch_rebases_offsets():
    from synth.families import sample_batch
    b = sample_batch(50, 20, 11)
    for rank in range(3):
        m0, m1, view, off, ln = local_batch(b.data, b.offsets, b.lengths, rank, 3)
        for k in range(m1 - m0):
            assert view[off[k]:off[k] + ln[k]].tobytes() == b.module(m0 + k)
            assert off[k] % 16 == 0


def _cpu_fn(view, off, ln):
    from oracle import disasm as odis
    texts = [odis.disassemble(view[o:o + n].tobytes()).encode() for o, n in zip(off, ln)]
    spans, pos, parts = [], 0, []
    for t in texts:
        spans.append((pos, len(t)))
        parts.append(t)
        pos += len(t)
    return np.frombuffer(b"".join(parts), dtype=np.uint8), np.array(spans, dtype=np.int64), \
        np.zeros(len(texts), np.int32)


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2305_09493_b200.shard import run_sharded
    from synth.families import sample_batch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b = sample_batch(40, 20, 5)
        m0, m1, arena, spans, status, base, totals = run_sharded(_cpu_fn, b.data, b.offsets, b.lengths)
        q.put((rank, m0, m1, arena.tobytes(), spans.tolist(), base, totals))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_run_sharded_gloo_world2():
    import torch.multiprocessing as mp
    from synth.families import sample_batch
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
    b = sample_batch(40, 20, 5)
    whole = _cpu_fn(b.data, b.offsets, b.lengths)
    arena = b"".join(r[3] for r in res)
    assert arena == whole[0].tobytes()
    assert res[0][1] == 0 and res[-1][2] == b.n and res[0][2] == res[1][1]
    assert res[0][6] == res[1][6] == [len(r[3]) for r in res]
    spans = [s for r in res for s in r[4]]
    assert spans == whole[1].tolist()          # global placement == single-process layout
    assert res[1][5] == len(res[0][3])


# -- bench.py: the config-5 sharded batch and the --gpus self-launch ---------------------
def _c5_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pool, pick, lengths, m0, m1 = bench.config5_shard(300, 25, rank, world, seed=7)
        pool_t = [torch.from_numpy(pool.data.copy()), torch.from_numpy(pool.offsets.astype(np.int64)),
                  torch.from_numpy(pool.lengths.astype(np.int64))]
        chunks = []
        for c0 in range(m0, m1, 64):      # device chunks, built here on CPU tensors
            b = bench.device_chunk(*pool_t, pick[c0:min(m1, c0 + 64)])
            off, ln = b.off.numpy(), b.len.numpy()
            chunks.append([b.data[o:o + n].numpy().tobytes() for o, n in zip(off, ln)])
        words = torch.tensor([int(lengths[m0:m1].sum()) // 4])
        dist.all_reduce(words)
        q.put((rank, m0, m1, [m for c in chunks for m in c], int(words.item())))
    finally:
        dist.destroy_process_group()


def test_config5_shard_gloo_world2():
    """Each rank builds only its own range of the one global batch; together the ranks
    cover it exactly, module bytes equal sample_batch's, and the all-reduced word count
    is the batch total."""
    import torch.multiprocessing as mp
    from synth.families import sample_batch
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_c5_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    whole = sample_batch(300, 25, 7)
    assert res[0][1] == 0 and res[0][2] == res[1][1] and res[1][2] == 300
    mods = res[0][3] + res[1][3]
    assert mods == [whole.module(i) for i in range(300)]
    assert res[0][4] == res[1][4] == whole.words


def test_bench_gpus_self_launch():
    """`bench.py --gpus 2` without torchrun relaunches itself with one process per rank
    (here the reference arm: rank 0 prints, the other rank exits 0)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--steps", "1", "--warmup", "3", "--cpu-per-core", "1", "--ref-modules", "50",
                          "--variants", "50"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2
