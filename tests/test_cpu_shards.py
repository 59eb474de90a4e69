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
from paper_2604_07239_b200.errors import FormatError, IntegrityError
from paper_2604_07239_b200.model import default_device
from paper_2604_07239_b200.shard import compress_sharded, decompress_sharded, shard_bounds


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


def fake_decompress(shard, fp):
    """Stand-in for the device decode of one shard (inverse of fake_compress)."""
    part = StreamPartition.from_length(shard.original_length, len(shard.stream_lengths))
    mat = np.frombuffer(shard.payload, np.uint8).reshape(len(shard.stream_lengths), -1)
    return part.join(mat)


def _worker(rank, world, port, data, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # one process per GPU: a rank's models land on its LOCAL_RANK device
        assert default_device() == rank
        cfg = ModelConfig(ctx_len=4, embed_dim=8, cache_dim=32, mix_dim=8, expand_dim=32,
                          batch=4, workers=1)
        blob = compress_sharded(data, cfg, compress_fn=fake_compress,
                                fingerprint_fn=lambda c: 0x1000 + rank)
        if rank == 0:
            with open(out, "wb") as fh:
                fh.write(blob)
        else:
            assert blob is None
        # every rank decodes its share of the shards; rank 0 joins them
        blob = open(out, "rb").read() if rank == 0 else None
        objs = [blob]
        dist.broadcast_object_list(objs, src=0)
        back = decompress_sharded(objs[0], decompress_fn=fake_decompress)
        if rank == 0:
            assert back == data
            with open(out + ".ok", "w") as fh:
                fh.write("ok")
        else:
            assert back is None
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
    assert open(out + ".ok").read() == "ok"
    shards = container.unpack_shards(blob)
    assert len(shards) == world
    assert [s.fingerprint for s, _ in shards] == [0x1000 + r for r in range(world)]
    # each shard's streams are the partition of its contiguous chunk
    joined = b""
    for (shard, _fp), (lo, hi) in zip(shards, shard_bounds(len(data), world)):
        assert shard.original_length == hi - lo
        part = StreamPartition.from_length(shard.original_length, len(shard.stream_lengths))
        mat = np.frombuffer(shard.payload, np.uint8).reshape(len(shard.stream_lengths), -1)
        joined += part.join(mat)
    assert joined == data


def _results(data, n):
    cfg = ModelConfig(ctx_len=4, embed_dim=8, cache_dim=32, mix_dim=8, expand_dim=32, batch=4,
                      workers=1)
    return cfg, [fake_compress(data[lo:hi], cfg) for lo, hi in shard_bounds(len(data), n)]


def test_v2_per_shard_crc_names_the_corrupt_shard():
    data = corpus.make_text(2000, 3)
    cfg, res = _results(data, 3)
    blob = bytearray(container.pack_shards(res, cfg, [7, 8, 9]))
    shards = container.unpack_shards(bytes(blob))
    # flip one byte inside shard 1's payload
    start = len(blob) - sum(len(s.payload) for s, _ in shards)
    pos = start + len(shards[0][0].payload) + 5
    blob[pos] ^= 0x40
    with pytest.raises(IntegrityError, match="shard 1"):
        container.unpack_shards(bytes(blob))
    with pytest.raises(IntegrityError):
        container.decompress_bytes(bytes(blob))


def test_v2_header_crc_and_inspect():
    data = corpus.make_text(1500, 4)
    cfg, res = _results(data, 2)
    blob = container.pack_shards(res, cfg, [0xAB, 0xCD])
    info = container.inspect_blob(blob)
    assert info["version"] == 2 and info["n_shards"] == 2 and info["checksums_ok"]
    assert info["original_length"] == len(data)
    assert [s["fingerprint"] for s in info["shards"]] == ["0x000000ab", "0x000000cd"]
    assert sum(s["original_length"] for s in info["shards"]) == len(data)
    bad = bytearray(blob)
    bad[100] ^= 1       # inside the shard table
    with pytest.raises((IntegrityError, FormatError)):
        container.inspect_blob(bytes(bad))
