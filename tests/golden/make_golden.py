"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run here (the container that has /root/reference); the outputs are committed
so the GPU box, which has no /root/reference, can use them:

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests \
        python tests/golden/make_golden.py

Every array in the .npz files is produced by the reference package ``dszip``
(numba backend) -- nothing here uses this repo's code, so the fixtures pin
both the oracle (tests/test_oracle.py) and the CUDA path (tests/test_gpu_*.py).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.path[:0] = ["/root/reference/pkg/src", "/root/reference/pkg/tests"]

import _corpus  # noqa: E402  (reference test corpus)
from dszip import container, kernels  # noqa: E402
from dszip.coder import BatchEncoder, cum_from_freq, quantize  # noqa: E402
from dszip.config import ModelConfig  # noqa: E402
from dszip.model import Predictor  # noqa: E402
from dszip.pipeline import run_serial_compress  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
NB = kernels.BACKENDS["numba"]


def softmax_rows(rng, rows, scale):
    lg = rng.normal(scale=scale, size=(rows, 256))
    p = np.exp(lg - lg.max(axis=1, keepdims=True))
    return p / p.sum(axis=1, keepdims=True)


def gen_quant():
    rng = np.random.default_rng(101)
    blocks = [softmax_rows(rng, 48, s) for s in (0.05, 0.5, 1.0, 2.0, 4.0, 10.0, 25.0)]
    near = np.full((8, 256), 1e-9)
    for k in range(8):
        near[k, (37 * k) % 256] = 1.0 - near[k].sum() + near[k, (37 * k) % 256]
    blocks.append(near)
    blocks.append(rng.dirichlet(np.ones(256) * 0.05, size=32))
    blocks.append(np.full((4, 256), 1.0 / 256))
    probs = np.ascontiguousarray(np.concatenate(blocks))
    freq = np.empty(probs.shape, np.int64)
    assert NB["quantize_rows"](probs, freq, 0, probs.shape[0]) == -1
    bad = probs[:3].copy()
    bad[0] *= 1.01      # sums > 1 -> deficit < 0
    bad[1] *= 0.99      # deficit > 256
    fb = np.empty(bad.shape, np.int64)
    bad_row = NB["quantize_rows"](bad, fb, 0, 3)
    np.savez_compressed(os.path.join(OUT, "quant.npz"), probs=probs, freq=freq,
                        bad_probs=bad, bad_row=np.int64(bad_row))


def gen_coder():
    """Bitstreams from the reference encoder for random tables (kernels.py:123-183)."""
    rng = np.random.default_rng(202)
    rows, steps = 32, 160
    cums = np.empty((steps, rows, 257), np.int64)
    syms = np.empty((steps, rows), np.int64)
    ucum = np.tile(np.arange(257, dtype=np.int64) * 256, (rows, 1))
    for i in range(steps):
        if i == 0:
            cums[i] = ucum      # real containers start every stream uniform-coded
        else:
            p = softmax_rows(rng, rows, rng.uniform(0.1, 6.0))
            f = np.empty((rows, 256), np.int64)
            assert NB["quantize_rows"](p, f, 0, rows) == -1
            cums[i] = cum_from_freq(f)
        # draw symbols mostly from the table, sometimes rare symbols
        f = np.diff(cums[i], axis=1)
        for k in range(rows):
            if rng.random() < 0.1:
                syms[i, k] = int(np.argmin(f[k]))
            else:
                syms[i, k] = rng.choice(256, p=f[k] / 65536.0)
    enc = BatchEncoder(rows)
    for i in range(steps):
        enc.encode(cums[i], syms[i], step=i)
    streams = enc.finish()
    lengths = np.array([len(s) for s in streams], np.int64)
    payload = np.frombuffer(b"".join(streams), np.uint8)

    # the first-byte 0xFF quirk: non-uniform first symbol
    qrows = 8
    qcum = np.zeros((2, qrows, 257), np.int64)
    f = np.ones((qrows, 256), np.int64)
    f[:, 0] = 65536 - 255
    qcum[0] = cum_from_freq(f)
    qcum[1] = np.tile(np.arange(257, dtype=np.int64) * 256, (qrows, 1))
    qsym = np.array([[255] * qrows, list(range(qrows))], np.int64)
    qenc = BatchEncoder(qrows)
    for i in range(2):
        qenc.encode(qcum[i], qsym[i], step=i)
    qstreams = qenc.finish()
    np.savez_compressed(
        os.path.join(OUT, "coder.npz"), cums=cums.astype(np.uint32), syms=syms.astype(np.uint8), payload=payload,
        lengths=lengths, quirk_cums=qcum, quirk_syms=qsym,
        quirk_payload=np.frombuffer(b"".join(qstreams), np.uint8),
        quirk_lengths=np.array([len(s) for s in qstreams], np.int64))


def run_model(cfg, data, steps):
    """Drive the reference Predictor through the serial order (pipeline.py:211-223)."""
    from dszip.pipeline import StreamPartition
    part = StreamPartition.from_length(len(data), cfg.batch)
    mat = part.split(data)
    model = Predictor(cfg)
    probs, losses, alphas = [], [], []
    t = cfg.ctx_len
    for i in range(t, t + steps):
        pr = model.predict(mat[:, i - t:i])
        probs.append(pr)
        alphas.append(model.alpha_stats)
        losses.append(model.train_step(mat[:, i]))
    return model, mat, np.array(probs), np.array(losses), np.array(alphas)


def gen_model(name, cfg, data, steps):
    model, mat, probs, losses, alphas = run_model(cfg, data, steps)
    st = model.save_state()
    t = cfg.ctx_len
    i = t + steps
    ctx = np.ascontiguousarray(mat[:, i - t:i])
    tgt = mat[:, i].astype(np.int64)
    parts = model.forward_debug(ctx)
    loss, grads = model.loss_grads(ctx, tgt)
    next_probs = model.predict(ctx)
    arrays = {"mat": mat[:, :i + 1], "probs": probs, "losses": losses, "alphas": alphas,
              "ctx": ctx, "tgt": tgt, "next_probs": next_probs, "gloss": np.float64(loss),
              "cache": st["cache"], "t": np.int64(st["t"]), "step_count": np.int64(st["step_count"])}
    for k, v in st["params"].items():
        arrays["p_" + k] = v
    for j, k in enumerate(st["params"]):
        arrays["m_" + k] = st["m"][j]
        arrays["v_" + k] = st["v"][j]
    for k, v in parts.items():
        arrays["part_" + k] = v
    for k, v in grads.items():
        arrays["g_" + k] = v
    # one more full train step from the saved state: params after update
    model.train_step(tgt)
    for k, v in model.params.items():
        arrays["next_p_" + k] = v.data
    arrays["next_cache"] = model.cache
    cfgd = {f: getattr(cfg, f) for f in ("ctx_len", "embed_dim", "cache_dim", "mix_dim",
                                          "expand_dim", "batch", "conv_kernel", "lr", "beta1",
                                          "beta2", "adam_eps", "seed", "workers")}
    arrays["cfg_json"] = np.frombuffer(json.dumps(cfgd).encode(), np.uint8)
    np.savez_compressed(os.path.join(OUT, f"model_{name}.npz"), **arrays)


def gen_variants():
    """Ablation variants (model.py:39, 121-175): per-step probabilities, losses
    and router stats from the seeded init, then the loss gradients."""
    from dszip.model import VARIANTS
    from dszip.pipeline import StreamPartition
    cfg = ModelConfig(ctx_len=4, embed_dim=8, cache_dim=32, mix_dim=8, expand_dim=32,
                      batch=16, workers=1, seed=9)
    data = _corpus.make_text(16 * 200, 4)
    mat = StreamPartition.from_length(len(data), cfg.batch).split(data)
    t, steps = cfg.ctx_len, 12
    arrays = {"mat": mat[:, :t + steps + 1]}
    for v in VARIANTS:
        model = Predictor(cfg, v)
        probs, losses, alphas = [], [], []
        for i in range(t, t + steps):
            probs.append(model.predict(mat[:, i - t:i]))
            alphas.append(model.alpha_stats if model.alpha_stats is not None else (np.nan,) * 3)
            losses.append(model.train_step(mat[:, i]))
        i = t + steps
        ctx = np.ascontiguousarray(mat[:, i - t:i])
        loss, grads = model.loss_grads(ctx, mat[:, i].astype(np.int64))
        arrays[v + "__probs"] = np.array(probs)[:, :8].astype(np.float32)   # 8 of 16 rows
        arrays[v + "__losses"] = np.array(losses)
        arrays[v + "__alphas"] = np.array(alphas, dtype=np.float64)
        arrays[v + "__gloss"] = np.float64(loss)
        for k, g in grads.items():   # parameters a variant never touches: no gradient
            arrays[v + "__g_" + k] = (np.zeros_like(model.params[k].data) if g is None
                                      else np.asarray(g, dtype=np.float32))
    np.savez_compressed(os.path.join(OUT, "variants.npz"), **arrays)


def gen_default_digest():
    """Default config (24 M params) is too big to store: keep digests + slices."""
    cfg = ModelConfig(seed=5)
    model = Predictor(cfg)
    digest = {k: hashlib.sha256(v.data.tobytes()).hexdigest() for k, v in model.params.items()}
    data = _corpus.make_text(1 << 20, 12)
    from dszip.pipeline import StreamPartition
    mat = StreamPartition.from_length(len(data), cfg.batch).split(data)
    t = cfg.ctx_len
    probs, losses = [], []
    for i in range(t, t + 3):
        pr = model.predict(mat[:, i - t:i])
        probs.append(pr[:32])
        losses.append(model.train_step(mat[:, i]))
    sl = {k: v.data.reshape(-1)[:4096].copy() for k, v in model.params.items()}
    np.savez_compressed(os.path.join(OUT, "model_default_digest.npz"),
                        probs=np.array(probs), losses=np.array(losses),
                        **{"slice_" + k: v for k, v in sl.items()},
                        digest_json=np.frombuffer(json.dumps(digest).encode(), np.uint8))


def gen_container():
    """Reference containers and bits/byte at sizes the GPU tests re-run."""
    out = {}
    tiny = ModelConfig(ctx_len=4, embed_dim=8, cache_dim=32, mix_dim=8, expand_dim=32,
                       batch=16, workers=4, seed=11)
    # warm-up-only inputs: no model step, so the bytes are bit-reproducible
    for n in (0, 1, 5, 63, 64, 200):
        data = _corpus.make_text(n, 3) if n else b""
        blob, _ = container.compress_bytes(data, tiny)
        out[f"warm_{n}"] = np.frombuffer(blob, np.uint8)
    sizes = {}
    cases = {
        "tiny_text16k": (tiny, "text", 16384, 4),
        "mid_text64k": (ModelConfig(ctx_len=8, embed_dim=16, cache_dim=256, mix_dim=32,
                                    expand_dim=256, batch=64, workers=1, seed=6),
                        "text", 65536, 12),
        "mid_dna64k": (ModelConfig(ctx_len=8, embed_dim=16, cache_dim=256, mix_dim=32,
                                   expand_dim=256, batch=64, workers=1, seed=6),
                       "dna", 65536, 3),
    }
    for name, (cfg, kind, n, seed) in cases.items():
        data = getattr(_corpus, "make_" + kind)(n, seed)
        res = run_serial_compress(data, cfg)
        blob = container._pack(res)
        sizes[name] = {"bytes": len(blob), "payload": int(sum(len(s) for s in res.streams)),
                       "n": n, "kind": kind, "seed": seed,
                       "mean_loss": float(np.mean(res.losses)),
                       "cfg": {f: getattr(res.cfg, f) for f in (
                           "ctx_len", "embed_dim", "cache_dim", "mix_dim", "expand_dim",
                           "batch", "conv_kernel", "seed", "workers")}}
    # measured in BASELINE.md (22 min per direction on 8 cores): crit-5 workload
    sizes["default_text1m"] = {"bytes": 233320, "payload": 229126, "n": 1 << 20,
                               "kind": "text", "seed": 12, "mean_loss": 1.16469,
                               "cfg": {"seed": 5}, "source": "BASELINE.md section 2"}
    np.savez_compressed(os.path.join(OUT, "containers.npz"), **out)
    with open(os.path.join(OUT, "bpb.json"), "w") as fh:
        json.dump(sizes, fh, indent=1, sort_keys=True)


def gen_corpus_digest():
    dig = {}
    for kind, n, seed in (("text", 100000, 12), ("text", 4096, 3), ("dna", 50000, 3),
                          ("records", 10000, 2), ("random", 5000, 1), ("mixed", 200000, 4),
                          ("text", 1 << 20, 12)):
        data = getattr(_corpus, "make_" + kind)(n, seed)
        dig[f"{kind}_{n}_{seed}"] = hashlib.sha256(data).hexdigest()
    with open(os.path.join(OUT, "corpus_digest.json"), "w") as fh:
        json.dump(dig, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["quant", "coder", "model", "container", "corpus", "default",
                             "variants"]
    if "quant" in which:
        gen_quant()
    if "coder" in which:
        gen_coder()
    if "corpus" in which:
        gen_corpus_digest()
    if "model" in which:
        tiny = ModelConfig(ctx_len=4, embed_dim=8, cache_dim=32, mix_dim=8, expand_dim=32,
                           batch=16, workers=1, seed=9)
        gen_model("tiny", tiny, _corpus.make_text(16 * 200, 4), 40)
        mid = ModelConfig(ctx_len=8, embed_dim=16, cache_dim=256, mix_dim=32, expand_dim=256,
                          batch=64, workers=1, seed=6)
        gen_model("mid", mid, _corpus.make_text(64 * 200, 12), 30)
    if "container" in which:
        gen_container()
    if "variants" in which:
        gen_variants()
    if "default" in which:
        gen_default_digest()
    print("golden fixtures written to", OUT)
