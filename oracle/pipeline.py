"""TEST INFRASTRUCTURE ONLY: serial executor over the CPU oracle.

Restates ``pkg/src/dszip/pipeline.py:197-226`` (serial compress) and
``:310-396`` (decompress, single worker) on top of ``oracle.model`` and
``oracle.coder``.  Used by tests as a small-size checker and by bench.py as the
timed CPU baseline (the reference itself cannot travel to the GPU box).
"""

from __future__ import annotations

import time

import numpy as np

from . import coder as oc
from .model import OracleModel


def partition(data: bytes, b: int):
    length = -(-len(data) // b) if data else 0
    flat = np.zeros(b * length, dtype=np.uint8)
    flat[:len(data)] = np.frombuffer(data, dtype=np.uint8)
    return flat.reshape(b, length)


def compress(data: bytes, cfg):
    """Returns (streams, losses) of the reference's serial order."""
    mat = partition(data, cfg.batch)
    steps = mat.shape[1]
    warm = min(cfg.ctx_len, steps)
    model = OracleModel(cfg) if steps > warm else None
    enc = oc.Encoder(cfg.batch, steps)
    ucum = oc.uniform_cum(cfg.batch)
    losses = []
    for i in range(steps):
        if i < warm:
            cum = ucum
        else:
            cum = oc.cum_from_freq(oc.quantize(model.predict(mat[:, i - cfg.ctx_len:i])))
        enc.encode(cum, mat[:, i].astype(np.int64))
        if i >= warm:
            losses.append(model.train_step(mat[:, i]))
    return enc.finish(), losses


def time_steps(cfg, steps: int, warmup: int = 1, seed: int = 0):
    """Seconds per timestep of predict -> quantise -> encode -> train on random
    context (per-step cost does not depend on content)."""
    rng = np.random.default_rng(seed)
    model = OracleModel(cfg)
    enc = oc.Encoder(cfg.batch, steps + warmup + 1)
    times = []
    for k in range(warmup + steps):
        ctx = rng.integers(0, 256, size=(cfg.batch, cfg.ctx_len), dtype=np.uint8)
        tgt = rng.integers(0, 256, size=cfg.batch, dtype=np.uint8)
        t0 = time.perf_counter()
        cum = oc.cum_from_freq(oc.quantize(model.predict(ctx)))
        enc.encode(cum, tgt.astype(np.int64))
        model.train_step(tgt)
        if k >= warmup:
            times.append(time.perf_counter() - t0)
    return times
