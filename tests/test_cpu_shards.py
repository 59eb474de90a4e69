"""Multi-rank (world_size 2, gloo, CPU) coverage of the sharded path's host
logic: shard bounds, per-rank compress call, gather into a v2 container, and
the sharded decode fan-out.  The per-shard device compress is replaced by a
deterministic stand-in here (no GPU in this container); the GPU test
tests/test_gpu_roundtrip.py covers the device path per shard."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_07239_b200 import ModelConfig, container, corpus
from paper_2604_07239_b200.pipeline import CompressResult, StreamPartition
from paper_2604_07239_b200.shard import compress_sharded, shard_bounds


def test_shard_bounds_cover_input():
    for n, w in ((0, 2), (1, 4), (10, 3), (1000, 8), (7, 7)):
        b = shard_bounds(n, w)
        assert len(b) == w and b[0][0] == 0 and b[-1][1] == n
        assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
        sizes = [hi - lo for lo, hi in b]
        assert max(sizes) - min(sizes) <= 1


def fake_compress(data, cfg):
    """Stand-in for the device compress: streams = raw partition rows."""
    cfg = cfg.shrink_to_fit(len(data))
    part = StreamPartition.from_length(len(data), cfg.batch)
    mat = part.split(data) if data else np.zeros((cfg.batch, 0), np.uint8)
    return CompressResult([mat[k].tobytes() for k in range(cfg.batch)], cfg, part, [0.0])


def _worker(rank, world, port, data, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = ModelConfig(ctx_len=4, embed_dim=8, cache_dim=32, mix_dim=8, expand_dim=32,
                          batch=4, workers=1)
        blob = compress_sharded(data, cfg, compress_fn=fake_compress)
        if rank == 0:
            with open(out, "wb") as fh:
                fh.write(blob)
        else:
            assert blob is None
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2])
def test_gather_into_v2_container(tmp_path, world):
    data = corpus.make_text(3001, 9)
    out = str(tmp_path / "blob")
    mp.spawn(_worker, args=(world, _free_port(), data, out), nprocs=world, join=True)
    blob = open(out, "rb").read()
    shards = container.unpack_shards(blob)
    assert len(shards) == world
    # each shard's streams are the partition of its contiguous chunk
    joined = b""
    for (shard, _fp), (lo, hi) in zip(shards, shard_bounds(len(data), world)):
        assert shard.original_length == hi - lo
        part = StreamPartition.from_length(shard.original_length, len(shard.stream_lengths))
        mat = np.frombuffer(shard.payload, np.uint8).reshape(len(shard.stream_lengths), -1)
        joined += part.join(mat)
    assert joined == data
