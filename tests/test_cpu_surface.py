"""CPU-only checks of the host side: corpus restatement, container layout,
config semantics, partitioning, the ABI library's exports, and the sharded
container writer."""

import ctypes
import hashlib
import os
import re
import struct
import zlib

import numpy as np
import pytest

from conftest import ROOT, golden_json, load_golden
from paper_2604_07239_b200 import ModelConfig, UsageError, container, corpus
from paper_2604_07239_b200.errors import FormatError, IntegrityError
from paper_2604_07239_b200.pipeline import CompressResult, PingPongBuffer, StreamPartition


@pytest.mark.parametrize("key", sorted(golden_json("corpus_digest.json")))
def test_corpus_matches_reference(key):
    kind, n, seed = key.split("_")
    data = getattr(corpus, "make_" + kind)(int(n), int(seed))
    assert hashlib.sha256(data).hexdigest() == golden_json("corpus_digest.json")[key]


def test_floats_and_modal_generators():
    f = corpus.make_floats(4000, 3)
    assert len(f) == 4000 and f == corpus.make_floats(4000, 3)
    m = corpus.make_modal(30, 1, chunk=10)
    assert len(m) == 30 and set(m[10:20]) <= set(b"ACGT")


class TestConfig:
    def test_defaults_and_hidden(self):
        c = ModelConfig()
        assert (c.ctx_len, c.embed_dim, c.cache_dim, c.batch, c.hidden_dim) == (16, 32, 4096, 512, 512)

    def test_validate_rejects(self):
        for bad in (dict(conv_kernel=2), dict(cache_dim=33), dict(workers=3), dict(lr=0.0),
                    dict(alphabet=255), dict(batch=0)):
            with pytest.raises(UsageError):
                ModelConfig(**bad).validate()

    def test_shrink_to_fit(self):
        c = ModelConfig(batch=512, workers=8).shrink_to_fit(100)
        assert c.batch * c.ctx_len <= 100 or c.batch == 1
        assert c.batch % c.workers == 0
        assert ModelConfig().shrink_to_fit(1 << 20) == ModelConfig()

    def test_device_check(self):
        with pytest.raises(UsageError):
            ModelConfig(embed_dim=6, cache_dim=60).device_check()
        ModelConfig().device_check()


def test_partition_round_trip():
    part = StreamPartition.from_length(1000, 16)
    assert (part.stream_length, part.pad) == (63, 16 * 63 - 1000)
    data = bytes(range(256)) * 4
    mat = part.split(data[:1000])
    assert mat.shape == (16, 63) and part.join(mat) == data[:1000]
    assert (mat[0, :63] == np.frombuffer(data[:63], np.uint8)).all()


def test_pingpong_protocol_trace():
    """Replaying a device event tape: warm-up steps first, then the model
    steps in device-time order; every slot follows the legal cycle."""
    seen = []
    # two model steps after 2 warm-up steps; step 3 fills while 2 still drains?
    # no: the model stream waits for the drain of step i before step i+1
    tape = np.array([[100, 110, 111, 115, 130],
                     [131, 140, 141, 144, 160]], np.int64)
    ev = PingPongBuffer(seen.append).replay_tape(2, tape)
    assert seen[:4] == [(0, "empty", "filling"), (0, "filling", "full"),
                        (0, "full", "draining"), (0, "draining", "empty")]
    assert len(seen) == 16
    assert [e[1] for e in ev[8:]] == [2] * 4 + [3] * 4
    assert [s for s, _, _ in seen[8:12]] == [0] * 4 and [s for s, _, _ in seen[12:]] == [1] * 4


def test_pingpong_rejects_an_illegal_tape():
    """A tape where slot 0 is refilled before it drained fails the reference's
    transition check (pipeline.py:78-83)."""
    tape = np.array([[100, 110, 150, 160, 170],
                     [120, 125, 126, 127, 128],
                     [130, 135, 136, 137, 138]], np.int64)   # step 2 (slot 0) fills at 130 < 150
    with pytest.raises(AssertionError):
        PingPongBuffer().replay_tape(0, tape)


def test_product_init_matches_reference_default_digest():
    """The product's seeded draw (model.init_params, uploaded by every
    Predictor) equals the reference's default-config init byte for byte."""
    import hashlib
    import json
    from paper_2604_07239_b200.config import ModelConfig
    from paper_2604_07239_b200.model import PARAM_ORDER, init_params
    z = load_golden("model_default_digest.npz")
    dig = json.loads(bytes(z["digest_json"]).decode())
    p = init_params(ModelConfig(seed=5))
    for k in PARAM_ORDER:
        assert hashlib.sha256(p[k].tobytes()).hexdigest() == dig[k], k


class TestContainer:
    def test_reference_warm_containers_parse(self):
        z = load_golden("containers.npz")
        for key in z.files:
            blob = z[key].tobytes()
            info, payload = container.unpack_header(blob)
            assert info.version == 1
            assert len(blob) == container.header_size(len(info.stream_lengths)) + len(payload)
            n = int(key.split("_")[1])
            assert info.original_length == n

    def test_header_layout_matches_reference(self):
        # repack a reference blob's streams with our writer: identical bytes except the
        # build fingerprint (offset 82) and the header CRC that covers it
        z = load_golden("containers.npz")
        blob = z["warm_200"].tobytes()
        info, payload = container.unpack_header(blob)
        lens = info.stream_lengths
        offs = np.concatenate([[0], np.cumsum(lens)])
        streams = [payload[offs[k]:offs[k + 1]] for k in range(len(lens))]
        part = StreamPartition.from_length(info.original_length, len(lens))
        ours = container._pack(CompressResult(streams, info.cfg, part))
        head = container.header_size(len(lens)) - 8
        assert ours[:82] == blob[:82]
        assert ours[90:head] == blob[90:head]
        assert ours[-len(payload):] == payload
        assert ours[head + 4:head + 8] == blob[head + 4:head + 8]   # payload crc

    def test_empty_container_is_98_bytes(self):
        blob = container._pack(CompressResult([], ModelConfig(batch=4, workers=1),
                                              StreamPartition.from_length(0, 4)))
        assert len(blob) == 98
        assert container.decompress_bytes(blob) == b""

    def test_rejections(self):
        z = load_golden("containers.npz")
        blob = bytearray(z["warm_64"].tobytes())
        with pytest.raises(FormatError):
            container.unpack_header(b"FAD")
        bad = bytearray(blob)
        bad[0:4] = b"NOPE"
        with pytest.raises(FormatError):
            container.unpack_header(bytes(bad))
        bad = bytearray(blob)
        bad[-1] ^= 0xFF
        with pytest.raises(IntegrityError):
            container.unpack_header(bytes(bad))
        bad = bytearray(blob)
        struct.pack_into("<H", bad, 4, 9)
        with pytest.raises(FormatError):
            container.unpack_header(bytes(bad))

    def test_sharded_round_trip_of_tables(self):
        cfg = ModelConfig(batch=4, workers=1)
        res = []
        for k in range(3):
            streams = [bytes([k, j]) * (j + 2) for j in range(4)]
            res.append(CompressResult(streams, cfg, StreamPartition.from_length(10 + k, 4)))
        blob = container.pack_shards(res, cfg, [1, 2, 3])
        shards = container.unpack_shards(blob)
        assert [s.original_length for s, _ in shards] == [10, 11, 12]
        assert shards[2][0].payload == b"".join(res[2].streams)
        bad = bytearray(blob)
        bad[-1] ^= 1
        with pytest.raises(IntegrityError):
            container.unpack_shards(bytes(bad))

    def test_scores(self):
        assert container.compression_ratio(100, 50) == 2.0
        assert container.compression_ratio(0, 5) == 0.0
        assert container.weighted_score(2, 10, 1, 3, 0, 20) == pytest.approx(0.5)


def test_abi_library_exports_every_declared_symbol():
    from paper_2604_07239_b200 import _native
    header = open(os.path.join(ROOT, "include", "fade_b200.h")).read()
    declared = set(re.findall(r"FADE_API\s+[\w\s\*]+?\b(fade_\w+)\s*\(", header))
    assert len(declared) >= 25
    so = ctypes.CDLL(_native.LIB_PATH)       # loads without a GPU (static cudart)
    missing = [s for s in declared if not hasattr(so, s)]
    assert not missing
    assert declared == set(_native.SIGNATURES)
    assert so.fade_abi_version() == 3


def test_active_params_match_reference_gradients():
    """Each variant's active parameter set (model.active_params) is exactly the
    set of tensors the reference gives a gradient (tests/golden/variants.npz
    stores zeros where the reference had none)."""
    from conftest import load_golden
    from paper_2604_07239_b200.model import PARAM_ORDER, VARIANTS, active_params
    z = load_golden("variants.npz")
    for v in VARIANTS:
        reached = {n for n in PARAM_ORDER if np.abs(z[v + "__g_" + n]).max() > 0}
        assert set(active_params(v)) == reached, v


def test_order0_entropy():
    from paper_2604_07239_b200 import harness
    assert harness.order0_entropy(bytes(range(256)) * 4) == pytest.approx(8.0)
    assert harness.order0_entropy(b"\x00" * 100) == 0.0
    assert harness.order0_entropy(b"") == 0.0
