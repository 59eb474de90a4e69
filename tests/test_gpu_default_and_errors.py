"""The shipped geometry pinned to the reference, and the device error paths.

* ``ModelConfig(seed=5)`` (B = 512, the bench configuration: the specialised
  trunk kernels, the X = 128 fused W_U Adam path of bmm_bwd, CTA-pair and
  persistent GEMMs, the default split plans) for three online steps from the
  seeded init on the criterion-5 text, against the reference's own
  probabilities and losses (tests/golden/model_default_digest.npz, written by
  running dszip itself in tests/golden/make_golden.py:192-210).  Tolerances as
  tests/test_gpu_model.py states them (TF32 operand truncation).
* ``ModelDivergenceError.step`` is the model's ``step_count`` (ref
  model.py:190-193, 208-209), not the coder column, for the Predictor API and
  for the executors; a failed predict leaves the cache as it was.
* The decoder's invalid-code path (why = 1, ref kernels.py:205-206,
  coder.py:124-128) raised by the device executor and the kernel table.
"""

import ctypes

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def kl_bits(p, q):
    return float(np.mean(np.sum(p * (np.log2(p) - np.log2(q)), axis=1)))


def tiny(**kw):
    from paper_2604_07239_b200 import ModelConfig
    base = dict(ctx_len=4, embed_dim=8, cache_dim=32, mix_dim=8, expand_dim=32, batch=16,
                workers=4, seed=11)
    base.update(kw)
    return ModelConfig(**base)


def test_default_geometry_matches_reference_digest():
    from paper_2604_07239_b200 import ModelConfig, corpus
    from paper_2604_07239_b200.model import Predictor
    from paper_2604_07239_b200.pipeline import StreamPartition
    z = load_golden("model_default_digest.npz")
    cfg = ModelConfig(seed=5)
    data = corpus.make_text(1 << 20, 12)
    mat = StreamPartition.from_length(len(data), cfg.batch).split(data)
    m = Predictor(cfg)
    t = cfg.ctx_len
    for j in range(z["probs"].shape[0]):
        i = t + j
        p = m.predict(mat[:, i - t:i])
        ref = z["probs"][j]
        got = p[:ref.shape[0]]
        assert np.abs(got - ref).max() < 1e-3, (j, float(np.abs(got - ref).max()))
        assert kl_bits(ref, got) < 1e-6, (j, kl_bits(ref, got))
        loss = m.train_step(mat[:, i])
        assert abs(loss - float(z["losses"][j])) < 1e-3 * float(z["losses"][j]), (j, loss)
    # the first 4096 elements of every parameter after the three updates
    s = m.save_state()["params"]
    for k, v in s.items():
        ref = z["slice_" + k]
        got = v.reshape(-1)[:ref.size]
        assert np.abs(got - ref).max() <= 2.5 * cfg.lr * 3, k


def _nan_state(m):
    st = m.save_state()
    st["params"] = dict(st["params"])
    st["params"]["w_head"] = np.full_like(st["params"]["w_head"], np.nan)
    return st


def test_predict_divergence_reports_step_count_and_keeps_cache():
    from paper_2604_07239_b200.errors import ModelDivergenceError
    from paper_2604_07239_b200.model import Predictor
    cfg = tiny()
    m = Predictor(cfg)
    rng = np.random.default_rng(0)
    for _ in range(3):   # three clean steps: step_count = 3
        m.predict(rng.integers(0, 256, (cfg.batch, cfg.ctx_len), dtype=np.uint8))
        m.train_step(rng.integers(0, 256, cfg.batch, dtype=np.uint8))
    st = _nan_state(m)
    st["step_count"] = 7
    m.load_state(st)
    cache = m.save_state()["cache"]
    with pytest.raises(ModelDivergenceError) as ei:
        m.predict(rng.integers(0, 256, (cfg.batch, cfg.ctx_len), dtype=np.uint8))
    assert ei.value.step == 7
    np.testing.assert_array_equal(m.save_state()["cache"], cache)


@pytest.mark.parametrize("step_count", [0, 5])
def test_executor_divergence_reports_step_count(step_count):
    """fade_compress on a model whose head is NaN: the first model column is
    `warm`, and the error carries step_count (= column - warm + the model's
    starting count), as Predictor.predict raises it inside the reference loop."""
    from paper_2604_07239_b200 import _native, corpus
    from paper_2604_07239_b200.model import Predictor
    cfg = tiny()
    m = Predictor(cfg)
    st = _nan_state(m)
    st["step_count"] = step_count
    m.load_state(st)
    L = 40
    mat = np.frombuffer(corpus.make_text(cfg.batch * L, 2), np.uint8).reshape(cfg.batch, L).copy()
    lengths = np.zeros(cfg.batch, np.int64)
    coder = ctypes.c_void_p()
    err = _native.FadeError()
    rc = _native.lib().fade_compress(m.handle, m.device, cfg.batch, mat.ctypes.data, L,
                                     cfg.ctx_len, 0, 1, lengths.ctypes.data, None, None, None,
                                     ctypes.byref(coder), ctypes.byref(err))
    assert rc == 4 and err.kind == 4, (rc, _native.last_error())
    assert err.step == step_count
    assert not coder.value


def test_compress_bytes_divergence_raises():
    """An exploding learning rate diverges inside compress_bytes; the error
    names a step inside the run (step_count, never a column past it)."""
    from paper_2604_07239_b200 import container, corpus
    from paper_2604_07239_b200.errors import ModelDivergenceError
    data = corpus.make_text(4000, 3)
    cfg = tiny(lr=1e30)
    with pytest.raises(ModelDivergenceError) as ei:
        container.compress_bytes(data, cfg)
    L = -(-len(data) // cfg.batch)
    assert 0 <= ei.value.step < L - cfg.ctx_len


def test_decoder_invalid_code_why1_executor():
    """A stream whose first four bytes are FF FF FF FF primes code = 2^32 - 1,
    so dv = code // (range >> 16) = 65537 >= 65536 at the first symbol."""
    from paper_2604_07239_b200 import corpus
    from paper_2604_07239_b200.errors import CorruptionError
    from paper_2604_07239_b200.pipeline import run_parallel_decompress, run_pipelined_compress
    data = corpus.make_text(3000, 4)
    cfg = tiny()
    res = run_pipelined_compress(data, cfg)
    streams = [bytearray(s) for s in res.streams]
    streams[3][:4] = b"\xff\xff\xff\xff"
    lengths = np.array([len(s) for s in streams], np.int64)
    offsets = np.concatenate([[0], np.cumsum(lengths)[:-1]]).astype(np.int64)
    payload = np.frombuffer(b"".join(bytes(s) for s in streams), np.uint8)
    with pytest.raises(CorruptionError) as ei:
        run_parallel_decompress(payload, offsets, lengths, res.cfg, len(data))
    assert (ei.value.stream, ei.value.step) == (3, 0)
    assert "invalid code" in str(ei.value)


def test_decoder_invalid_code_why1_kernel_table():
    """The kernel-table decode_step (kernels.py:200-233 contract) returns
    (first failing row, why = 1) for the same primed code."""
    from paper_2604_07239_b200 import kernels
    n = 4
    # 8-byte streams (a symbol's renormalisation reads past the 4-byte prime);
    # stream 1 starts FF FF FF FF
    payload = np.frombuffer(b"\x00\x01\x02\x03" * 2 + b"\xff" * 8 + b"\x10\x20\x30\x40" * 2
                            + b"\x00" * 8, np.uint8)
    off = np.array([0, 8, 16, 24], np.int64)
    dlen = np.full(n, 8, np.int64)
    cum = np.tile((np.arange(257, dtype=np.int64) * 256)[None], (n, 1))
    pos, code, rng, out = (np.zeros(n, np.int64) for _ in range(4))
    be = kernels.BACKENDS["cuda"]
    assert be["prime"](payload, off, dlen, pos, code, rng, 0, n) == -1
    assert int(code[1]) == 0xFFFFFFFF
    k, why = be["decode_step"](cum, payload, off, dlen, pos, code, rng, out, 0, n)
    assert (k, why) == (1, 1)


def test_models_follow_the_requested_device():
    """Predictor / executors run on the device they are given and restore the
    caller's current device (everything used to land on GPU 0)."""
    import torch
    from paper_2604_07239_b200 import container, corpus
    from paper_2604_07239_b200.model import Predictor, default_device
    n = torch.cuda.device_count()
    last = n - 1
    torch.cuda.set_device(0)
    assert default_device() == 0
    m = Predictor(tiny(), device=last)
    assert m.device == last and torch.cuda.current_device() == 0
    data = corpus.make_text(2000, 7)
    blob, _ = container.compress_bytes(data, tiny(), device=last)
    assert torch.cuda.current_device() == 0
    assert container.decompress_bytes(blob, device=last) == data
    assert torch.cuda.current_device() == 0


def test_event_tape_orders_the_pingpong_protocol():
    """The trace callback sees the device's own slot transitions: per step,
    fill -> full -> drain -> empty with non-decreasing device timestamps,
    steps in order, and the metrics clock is the device tape."""
    from paper_2604_07239_b200 import corpus
    from paper_2604_07239_b200.pipeline import run_pipelined_compress
    data = corpus.make_text(3000, 9)
    seen = []
    res = run_pipelined_compress(data, tiny(), trace=seen.append, collect_metrics=True)
    L = -(-len(data) // res.cfg.batch)
    assert len(seen) == 4 * L
    per_slot = {0: [], 1: []}
    for slot, old, new in seen:
        per_slot[slot].append((old, new))
    for slot, tr in per_slot.items():
        cyc = [("empty", "filling"), ("filling", "full"), ("full", "draining"),
               ("draining", "empty")]
        assert tr == cyc * (len(tr) // 4)
    el = [r["elapsed_s"] for r in res.metrics]
    assert all(b > a for a, b in zip(el, el[1:])) and el[0] > 0


RING_CHECK = """
import sys
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
import test_gpu_default_and_errors as t
t._ring_check()
print("RING_OK")
"""


def test_ring_buffer_cache_tracks_the_oracle_roll():
    """The ring-buffer cache (experiments build, FADE_RING=1; off in the
    shipped library, engine.cu: measured slower) against the oracle's roll."""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    lib = os.path.join(ROOT, "build", "exp", "libfade_b200.so")
    if not os.path.exists(lib):
        pytest.skip("experiments build (make experiments) not present")
    env = dict(os.environ, FADE_LIB_PATH=lib, FADE_RING="1")
    code = RING_CHECK.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         timeout=600)
    assert "RING_OK" in out.stdout, out.stdout[-3000:] + out.stderr[-3000:]


def test_roll_cache_tracks_the_oracle_roll():
    """The shipped roll: same checks as the ring variant."""
    _ring_check()


def _ring_check():
    """D = 32, B = 64 runs the rolling cache as a block-major ring buffer (one
    block written per predict, the W_mem GEMMs rotate their TMA coordinates).  Over 20 steps
    (the 8-block ring wraps twice) the logical cache the device reports, the
    probabilities and the losses follow the CPU oracle's explicit roll
    (ref nn/ops.py:219-231); forward_debug and a failed predict leave the
    ring position untouched."""
    from oracle.model import OracleModel
    from paper_2604_07239_b200 import ModelConfig, corpus
    from paper_2604_07239_b200.model import Predictor
    cfg = ModelConfig(ctx_len=4, embed_dim=32, cache_dim=256, mix_dim=32, expand_dim=256,
                      batch=64, workers=1, seed=4)
    L = 30
    mat = np.frombuffer(corpus.make_text(cfg.batch * L, 5), np.uint8).reshape(cfg.batch, L)
    m, o = Predictor(cfg), OracleModel(cfg)
    T = cfg.ctx_len
    for i in range(T, T + 20):
        p = m.predict(mat[:, i - T:i])
        q = o.predict(mat[:, i - T:i])
        assert np.abs(p - q).max() < 2e-2, i
        if i == T + 9:
            before = m.save_state()["cache"]
            m.forward_debug(mat[:, i - T + 1:i + 1])
            np.testing.assert_array_equal(m.save_state()["cache"], before)
        np.testing.assert_allclose(m.save_state()["cache"], o.cache, atol=2e-2)
        lg, lr = m.train_step(mat[:, i]), o.train_step(mat[:, i])
        assert abs(lg - lr) < 2e-2, i
    # a cache set through the ABI reads back unchanged (ring reset to 0)
    st = m.save_state()
    st["cache"] = np.arange(cfg.batch * cfg.cache_dim, dtype=np.float32).reshape(cfg.batch, -1)
    m.load_state(st)
    np.testing.assert_array_equal(m.save_state()["cache"], st["cache"])


def test_warp_row_kernels_at_large_batch():
    """B >= 2048 runs the warp-per-row row kernels (row_warp.cu): probabilities
    and losses track the CPU oracle over a few online steps (H = 128 and 512
    instantiations), and a compress -> decompress round trip is lossless with
    the decoder replaying the encoder's losses bit for bit."""
    from oracle.model import OracleModel
    from paper_2604_07239_b200 import ModelConfig, corpus
    from paper_2604_07239_b200.model import Predictor
    from paper_2604_07239_b200.pipeline import run_parallel_decompress, run_pipelined_compress
    for dims in (dict(ctx_len=8, embed_dim=16, cache_dim=256, mix_dim=32, expand_dim=256),
                 dict(ctx_len=16, embed_dim=32, cache_dim=512, mix_dim=32, expand_dim=512)):
        cfg = ModelConfig(batch=2048, workers=1, seed=9, **dims)
        T = cfg.ctx_len
        L = T + 4
        mat = np.frombuffer(corpus.make_text(cfg.batch * L, 6), np.uint8).reshape(cfg.batch, L)
        m, o = Predictor(cfg), OracleModel(cfg)
        for i in range(T, T + 3):
            p, q = m.predict(mat[:, i - T:i]), o.predict(mat[:, i - T:i])
            assert np.abs(p - q).max() < 2e-3, (dims, i)
            lg, lr = m.train_step(mat[:, i]), o.train_step(mat[:, i])
            assert abs(lg - lr) < 2e-3 * max(1.0, abs(lr)), (dims, i)
    cfg = ModelConfig(batch=2048, workers=1, seed=9, ctx_len=8, embed_dim=16, cache_dim=256,
                      mix_dim=32, expand_dim=256)
    data = corpus.make_text(2048 * 24, 8)
    res = run_pipelined_compress(data, cfg)
    lengths = np.array([len(s) for s in res.streams], np.int64)
    offsets = np.concatenate([[0], np.cumsum(lengths)[:-1]]).astype(np.int64)
    out, losses = run_parallel_decompress(np.frombuffer(b"".join(res.streams), np.uint8), offsets,
                                          lengths, res.cfg, len(data), want_losses=True)
    assert out == data
    assert losses == res.losses


def test_schedule_is_deterministic_across_runs():
    """compute-sanitizer is closed on this GPU pool, so the three-stream PDL
    schedule is checked for races by its observable: the default-geometry
    kernels (B = 64) compress the same input to the same bytes three times,
    and the serial order (one stream, no overlap) writes the same container."""
    from paper_2604_07239_b200 import ModelConfig, container, corpus
    cfg = ModelConfig(batch=64, workers=1, seed=2)
    data = corpus.make_text(64 * 60, 3)
    blobs = [container.compress_bytes(data, cfg)[0] for _ in range(3)]
    assert blobs[0] == blobs[1] == blobs[2]
    assert container.compress_bytes(data, cfg, pipelined=False)[0] == blobs[0]
    assert container.decompress_bytes(blobs[0]) == data
