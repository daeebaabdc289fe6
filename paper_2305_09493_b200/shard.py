"""Multi-GPU batch sharding: one process per GPU, modules are
independent, so a batch is cut into contiguous module ranges balanced by bytes
and every rank runs the whole GPU path on its own range.  The only exchange is
a host-side all-gather of each shard's output byte total, which gives every
rank its global output offset; there is no collective on the data path.

The reference has no multi-process path (its API is one module per call,
``disasm.disassemble_module`` / ``asm.assemble_module``); these helpers only
partition a batch and place the shards' outputs in one global arena layout.
"""

from __future__ import annotations

import numpy as np


def shard_ranges(lengths, world: int) -> list[tuple[int, int]]:
    """Contiguous module ranges [m0, m1) for `world` ranks, split where the
    inclusive byte prefix sum crosses k/world of the total (empty ranges when
    there are fewer modules than ranks)."""
    lengths = np.asarray(lengths, dtype=np.int64)
    n = len(lengths)
    if world < 1:
        raise ValueError("world must be >= 1")
    cum = np.cumsum(lengths)
    total = int(cum[-1]) if n else 0
    cuts = [0]
    for k in range(1, world):
        # first module whose running byte total reaches k/world of the batch (integer
        # target ceil(total*k/world): same cut, no float conversion of cum per search)
        cut = int(np.searchsorted(cum, -(-total * k // world), side="left")) if total else n * k // world
        cuts.append(min(max(cut, cuts[-1]), n))
    cuts.append(n)
    return [(cuts[k], cuts[k + 1]) for k in range(world)]


def local_batch(data, offsets, lengths, rank: int, world: int):
    """(m0, m1, data view, offsets, lengths) of this rank's shard; offsets are
    rebased to the view (module starts keep their 16-byte alignment)."""
    offsets = np.asarray(offsets, dtype=np.int64)
    lengths = np.asarray(lengths, dtype=np.int64)
    m0, m1 = shard_ranges(lengths, world)[rank]
    if m1 <= m0:
        return m0, m1, np.zeros(16, dtype=np.uint8), offsets[:0], lengths[:0]
    b0 = int(offsets[m0])
    b1 = int((offsets[m1 - 1] + lengths[m1 - 1] + 15) // 16 * 16)
    view = np.asarray(data)[b0:max(b1, b0 + 16)]
    return m0, m1, view, offsets[m0:m1] - b0, lengths[m0:m1]


def gather_totals(local_total: int, group=None) -> list[int]:
    """All-gather one int64 per rank (host-side sizes; gloo or nccl)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([int(local_total)], dtype=torch.int64, device=dev)
    out = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return [int(x.item()) for x in out]


def place_shard(spans, local_total: int, group=None):
    """Global placement of this rank's output: returns (base, totals) where
    base = bytes of all lower ranks; spans (int64[n, 2], shard-relative) are
    shifted in place to global-arena offsets."""
    import torch.distributed as dist
    totals = gather_totals(local_total, group)
    base = sum(totals[: dist.get_rank(group)])
    if len(spans):
        spans[:, 0] += base
    return base, totals


def run_sharded(fn, data, offsets, lengths, group=None):
    """Run `fn(data, offsets, lengths) -> (arena uint8[], spans int64[n, 2],
    status int32[n])` on this rank's shard and place its output globally.

    Returns (m0, m1, arena, global spans, status, base, totals): this rank's
    modules are [m0, m1), its arena belongs at global byte `base` of an arena
    of sum(totals) bytes.  `fn` is the per-GPU path (e.g. a DisasmSession run).
    """
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    m0, m1, view, off, ln = local_batch(data, offsets, lengths, rank, world)
    if m1 > m0:
        arena, spans, status = fn(view, off, ln)
        spans = np.array(spans, dtype=np.int64).reshape(-1, 2)
    else:
        arena, spans, status = np.zeros(0, dtype=np.uint8), np.zeros((0, 2), np.int64), np.zeros(0, np.int32)
    base, totals = place_shard(spans, len(arena), group)
    return m0, m1, arena, spans, status, base, totals


def disasm_shard_fn(options=None, spec=None, ext=None):
    """The per-GPU disassembly path for run_sharded (host buffers in/out)."""
    from .disasm import DisasmSession
    sess = DisasmSession(options, spec, ext)

    def fn(view, off, ln):
        sess.stage(view, off, ln)
        text, spans, status = sess.run_staged()
        return text, spans, status
    return fn
