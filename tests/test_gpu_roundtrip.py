"""End-to-end on the B200: lossless round trips, serial == pipelined bytes,
decoder losses == encoder losses, warm-up-only containers bit-identical to the
reference's, and bits/byte within 0.5% of the reference's own containers."""

import numpy as np
import pytest

from conftest import golden_json, load_golden

pytestmark = pytest.mark.gpu


def tiny(**kw):
    from paper_2604_07239_b200 import ModelConfig
    base = dict(ctx_len=4, embed_dim=8, cache_dim=32, mix_dim=8, expand_dim=32, batch=16,
                workers=4, seed=11)
    base.update(kw)
    return ModelConfig(**base)


@pytest.mark.parametrize("kind,n", [("text", 3000), ("dna", 2000), ("records", 1500),
                                    ("random", 700), ("zeros", 900), ("mixed", 4000)])
def test_lossless(kind, n):
    from paper_2604_07239_b200 import container, corpus
    data = corpus.make_zeros(n) if kind == "zeros" else getattr(corpus, "make_" + kind)(n, 5)
    blob, _ = container.compress_bytes(data, tiny())
    assert container.decompress_bytes(blob) == data


@pytest.mark.parametrize("n", [0, 1, 5, 63, 64, 65, 200, 1001])
def test_tiny_and_ragged_inputs(n):
    from paper_2604_07239_b200 import container, corpus
    data = corpus.make_text(n, 3) if n else b""
    blob, res = container.compress_bytes(data, tiny())
    assert container.decompress_bytes(blob) == data


def test_warm_only_containers_match_reference_bytes():
    """No model step runs when L <= ctx_len: payload must equal the reference's."""
    from paper_2604_07239_b200 import container, corpus
    z = load_golden("containers.npz")
    checked = 0
    for key in z.files:
        n = int(key.split("_")[1])
        data = corpus.make_text(n, 3) if n else b""
        ours, _ = container.compress_bytes(data, tiny())
        assert container.decompress_bytes(ours) == data
        ref = z[key].tobytes()
        info, p_ref = container.unpack_header(ref)
        b = max(1, len(info.stream_lengths))
        length = -(-n // b) if n else 0
        if length > min(tiny().ctx_len, length):
            continue          # a model step ran: float trajectories differ by design
        _, p_ours = container.unpack_header(ours)
        assert p_ours == p_ref, key
        assert len(ours) == len(ref)
        checked += 1
    assert checked >= 3


def test_serial_equals_pipelined_and_losses_replay():
    from paper_2604_07239_b200 import container, corpus
    from paper_2604_07239_b200.pipeline import (run_parallel_decompress, run_pipelined_compress,
                                                run_serial_compress)
    data = corpus.make_text(6000, 7)
    a = run_serial_compress(data, tiny())
    b = run_pipelined_compress(data, tiny())
    assert a.streams == b.streams
    assert a.losses == b.losses
    lengths = np.array([len(s) for s in b.streams], dtype=np.int64)
    offsets = np.concatenate([[0], np.cumsum(lengths)[:-1]]).astype(np.int64)
    payload = np.frombuffer(b"".join(b.streams), np.uint8)
    out, losses = run_parallel_decompress(payload, offsets, lengths, b.cfg, len(data),
                                          want_losses=True)
    assert out == data
    assert losses == b.losses            # bit-identical float trajectory on both sides


@pytest.mark.parametrize("batch", [1, 200, 640])
def test_default_dims_at_ragged_stream_counts(batch):
    """Default model dims at stream counts that leave partial 128-row GEMM
    tiles (200, 640) or a single stream: lossless, and the decoder replays the
    encoder's losses bit for bit."""
    from paper_2604_07239_b200 import ModelConfig, corpus
    from paper_2604_07239_b200.pipeline import run_parallel_decompress, run_pipelined_compress
    data = corpus.make_text(batch * 40 if batch > 1 else 300, 9)
    res = run_pipelined_compress(data, ModelConfig(batch=batch, workers=1, seed=5))
    assert res.losses and all(np.isfinite(res.losses))
    lengths = np.array([len(s) for s in res.streams], dtype=np.int64)
    offsets = np.concatenate([[0], np.cumsum(lengths)[:-1]]).astype(np.int64)
    payload = np.frombuffer(b"".join(res.streams), np.uint8)
    out, losses = run_parallel_decompress(payload, offsets, lengths, res.cfg, len(data),
                                          want_losses=True)
    assert out == data
    assert losses == res.losses


def test_corrupt_payload_raises():
    from paper_2604_07239_b200 import CorruptionError, corpus
    from paper_2604_07239_b200.pipeline import run_parallel_decompress, run_serial_compress
    data = corpus.make_text(4000, 2)
    res = run_serial_compress(data, tiny())
    lengths = np.array([len(s) for s in res.streams], dtype=np.int64)
    offsets = np.concatenate([[0], np.cumsum(lengths)[:-1]]).astype(np.int64)
    payload = np.frombuffer(b"".join(res.streams), np.uint8)
    short = lengths.copy()
    short[3] = 5
    pay2 = np.concatenate([payload[o:o + n] for o, n in zip(offsets, short)])
    off2 = np.concatenate([[0], np.cumsum(short)[:-1]]).astype(np.int64)
    with pytest.raises(CorruptionError) as ei:
        run_parallel_decompress(pay2, off2, short, res.cfg, len(data))
    assert ei.value.stream == 3


def _bpb_case(name):
    from paper_2604_07239_b200 import ModelConfig, container, corpus
    case = golden_json("bpb.json")[name]
    cfg = ModelConfig(**case["cfg"])
    data = getattr(corpus, "make_" + case["kind"])(case["n"], case["seed"])
    blob, res = container.compress_bytes(data, cfg)
    assert container.decompress_bytes(blob) == data
    return len(blob), case["bytes"], res


@pytest.mark.parametrize("name", ["mid_text64k", "mid_dna64k", "tiny_text16k"])
def test_bits_per_byte_small(name):
    ours, ref, _ = _bpb_case(name)
    # small inputs: few hundred steps, so the statistical window is wider (2%)
    assert abs(ours - ref) / ref < 0.02, (ours, ref)


def test_bits_per_byte_default_1mib_within_half_percent():
    """Acceptance criterion 5 workload: default config, 1 MiB text, seed 5."""
    ours, ref, res = _bpb_case("default_text1m")
    rel = (ours - ref) / ref
    print(f"default 1 MiB: ours {ours} B vs reference {ref} B ({100 * rel:+.3f}%)")
    assert abs(rel) < 0.005, (ours, ref)


@pytest.mark.parametrize("kind", ["dna", "mixed"])
def test_bits_per_byte_default_1mib_dna_mixed(kind):
    """Beyond criterion 5: the reference's own containers for 1 MiB of DNA and
    mixed data at the default config (tests/golden/bpb_ref.jsonl, written by
    tests/golden/make_bpb_ref.py running dszip, ~25 min each on the CPU)."""
    import json
    import os
    from conftest import GOLDEN
    from paper_2604_07239_b200 import ModelConfig, container, corpus
    recs = [json.loads(l) for l in open(os.path.join(GOLDEN, "bpb_ref.jsonl"))]
    rec = next(r for r in recs if r["kind"] == kind)
    data = getattr(corpus, "make_" + kind)(rec["n"], rec["seed"])
    blob, _ = container.compress_bytes(data, ModelConfig(seed=5))
    assert container.decompress_bytes(blob) == data
    rel = (len(blob) - rec["bytes"]) / rec["bytes"]
    print(f"default 1 MiB {kind}: ours {len(blob)} B vs reference {rec['bytes']} B ({100 * rel:+.3f}%)")
    assert abs(rel) < 0.005, (len(blob), rec["bytes"])


def test_sharded_v2_container_round_trip():
    """independent shards (here run one after another on one GPU),
    host-side gather into a v2 container, decode back bit-exactly."""
    from paper_2604_07239_b200 import container, corpus
    from paper_2604_07239_b200.pipeline import run_pipelined_compress
    from paper_2604_07239_b200.shard import shard_bounds
    data = corpus.make_modal(9000, 2, chunk=3000)
    cfg = tiny()
    res = [run_pipelined_compress(data[lo:hi], cfg) for lo, hi in shard_bounds(len(data), 3)]
    blob = container.pack_shards(res, cfg)
    assert container.decompress_bytes(blob) == data


def test_metrics_tape_router_stats():
    """--metrics tape (pipeline.py:162-185): per-step loss and router alpha
    statistics from the device equal a host-driven predict/train_step replay
    (model.py:197-199), and the decoder's tape equals the encoder's."""
    from paper_2604_07239_b200 import corpus
    from paper_2604_07239_b200.model import Predictor
    from paper_2604_07239_b200.pipeline import (StreamPartition, run_parallel_decompress,
                                                run_pipelined_compress)
    data = corpus.make_text(3000, 9)
    cfg = tiny()
    res = run_pipelined_compress(data, cfg, collect_metrics=True)
    tape = res.metrics
    assert tape and all({"alpha_mean", "alpha_min", "alpha_max"} <= set(r) for r in tape)
    for r in tape:
        assert 0.0 <= r["alpha_min"] <= r["alpha_mean"] <= r["alpha_max"] <= 1.0
    # host replay of the first steps through the Predictor API
    part = StreamPartition.from_length(len(data), res.cfg.batch)
    mat = part.split(data)
    m = Predictor(res.cfg)
    T = res.cfg.ctx_len
    for k in range(4):
        i = T + k
        m.predict(mat[:, i - T:i])
        loss = m.train_step(mat[:, i])
        a = m.alpha_stats
        rec = tape[k]
        assert rec["step"] == i
        assert abs(rec["loss_nats"] - loss) < 1e-9
        assert abs(rec["alpha_mean"] - a[0]) < 1e-6
        assert rec["alpha_min"] == a[1] and rec["alpha_max"] == a[2]
    lengths = np.array([len(s) for s in res.streams], dtype=np.int64)
    offsets = np.concatenate([[0], np.cumsum(lengths)[:-1]]).astype(np.int64)
    payload = np.frombuffer(b"".join(res.streams), np.uint8)
    out, dtape = run_parallel_decompress(payload, offsets, lengths, res.cfg, len(data),
                                         collect_metrics=True)
    assert out == data
    assert [(r["loss_nats"], r["alpha_mean"], r["alpha_min"], r["alpha_max"]) for r in dtape] == \
        [(r["loss_nats"], r["alpha_mean"], r["alpha_min"], r["alpha_max"]) for r in tape]


def test_file_helpers_and_metrics_jsonl(tmp_path):
    """container.compress_file / decompress_file / inspect_file (the CLI's
    backing calls, container.py:186-220): report keys, lossless files, and the
    --metrics JSONL tape with device-clock elapsed_s."""
    import json
    from paper_2604_07239_b200 import container, corpus
    data = corpus.make_text(5000, 2)
    src, dst, back, met = (tmp_path / n for n in ("in", "out.fade", "back", "m.jsonl"))
    src.write_bytes(data)
    rep = container.compress_file(src, dst, tiny(), metrics_path=met)
    assert {"original_bytes", "compressed_bytes", "ratio", "bits_per_byte", "seconds",
            "kb_per_min", "n_streams", "pipelined"} <= set(rep)
    assert rep["compressed_bytes"] == dst.stat().st_size
    recs = [json.loads(l) for l in met.read_text().splitlines()]
    assert recs and all(r["phase"] == "compress" for r in recs)
    assert all(b["elapsed_s"] > a["elapsed_s"] for a, b in zip(recs, recs[1:]))
    rep2 = container.decompress_file(dst, back)
    assert back.read_bytes() == data and rep2["original_bytes"] == len(data)
    info = container.inspect_file(dst)
    assert info["version"] == 1 and info["checksums_ok"] and info["original_length"] == len(data)
