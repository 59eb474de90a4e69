"""Multi-GPU compression: independent chunk shards, one process per GPU.

SURVEY.md section 8e: the input is cut into G contiguous chunks; every rank
compresses its chunk with its own model and B streams on its own device (no
collective on the hot path).  The only exchange is host-side: rank 0 gathers
each shard's stream table and bytes and writes one v2 container
(`container.pack_shards`).  Decompression is equally independent: any rank can
decode any shard.

`torch.distributed` is plumbing here (object gather over gloo or NCCL); the
compute is the per-rank `run_pipelined_compress` on the rank's device.
"""

from __future__ import annotations

from dataclasses import replace

from .config import ModelConfig


def shard_bounds(n: int, world: int) -> list[tuple[int, int]]:
    """Contiguous [lo, hi) byte ranges, sizes differing by at most one."""
    base, extra = divmod(n, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def compress_shard(data: bytes, cfg: ModelConfig, rank: int, world: int, compress_fn=None,
                   device: int | None = None):
    """Compress this rank's chunk on ``device`` (default: this rank's
    ``model.default_device()``, i.e. LOCAL_RANK); returns its CompressResult."""
    from .pipeline import run_pipelined_compress
    lo, hi = shard_bounds(len(data), world)[rank]
    if compress_fn is not None:
        return compress_fn(data[lo:hi], cfg)
    return run_pipelined_compress(data[lo:hi], cfg, device=device)


def compress_sharded(data: bytes, cfg: ModelConfig, group=None, compress_fn=None,
                     device: int | None = None, fingerprint_fn=None,
                     local: bool = False) -> bytes | None:
    """Collective entry point: every rank calls it with the same `data`
    (``local=True``: each rank passes only its own contiguous shard, in rank
    order, so no rank needs the whole input in memory).

    Returns the v2 container on rank 0 and None elsewhere.  Each rank runs
    its shard on ``device`` (default: its own LOCAL_RANK GPU) and stamps it
    with its own ``shard_fingerprint`` (build + GPU architecture).
    """
    import torch.distributed as dist

    from . import container
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if local:
        res = compress_shard(data, cfg, 0, 1, compress_fn, device)
    else:
        res = compress_shard(data, cfg, rank, world, compress_fn, device)
    fp_fn = fingerprint_fn or (lambda c: container.shard_fingerprint(c, res.device or 0))
    # host-side gather of (stream table, bytes) -- the only exchange step
    payload = (res.partition.original_length, res.cfg, [bytes(s) for s in res.streams], res.losses,
               fp_fn(res.cfg))
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(payload, gathered, dst=0, group=group)
    if rank != 0:
        return None
    from .pipeline import CompressResult, StreamPartition
    results, fps = [], []
    for orig, rcfg, streams, losses, fp in gathered:
        rcfg = rcfg or replace(cfg, batch=max(1, len(streams)))
        results.append(CompressResult(streams, rcfg, StreamPartition.from_length(orig, len(streams)),
                                      losses))
        fps.append(fp)
    return container.pack_shards(results, cfg, fps)


def decompress_sharded(blob: bytes, group=None, device: int | None = None,
                       decompress_fn=None) -> bytes | None:
    """Each rank decodes its share of the shards on its own device; rank 0
    returns the bytes."""
    import torch.distributed as dist

    from . import container
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    shards = container.unpack_shards(blob)
    fn = decompress_fn or (lambda s, fp: container.decompress_shard(s, fp, device=device))
    mine = {i: fn(s, fp) for i, (s, fp) in enumerate(shards) if i % world == rank}
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(mine, gathered, dst=0, group=group)
    if rank != 0:
        return None
    parts = {}
    for g in gathered:
        parts.update(g)
    return b"".join(parts[i] for i in range(len(shards)))
