"""The online-trained byte predictor, resident on the B200.

``Predictor`` keeps the reference surface (``pkg/src/dszip/model.py:44-284``):
``predict``, ``train_step``, ``forward_debug``, ``eval_loss``, ``loss_grads``,
``save_state`` / ``load_state``, ``param_count`` and ``alpha_stats``.  All
parameters, Adam moments, the rolling cache and activations live on the device
(one ``fade_model_t``); the host only draws the seeded initialisation with
numpy exactly as the reference does (model.py:62-105) and uploads it.

All six variants of ``VARIANTS`` (model.py:39, 121-175) run on the device: the
ablations skip whole kernels and GEMMs.  As in the
reference, the container stores no variant and the decoder always rebuilds
``full`` (pipeline.py:329), so only ``full`` containers decode.
"""

from __future__ import annotations

import ctypes
import math
import os
import sys

import numpy as np

from . import _native
from .config import ModelConfig
from .errors import ModelDivergenceError, UsageError

VARIANTS = ("full", "dual", "global_only", "local_only", "mixer_nogate", "mixer")
LN2 = math.log(2.0)

PARAM_ORDER = (
    "emb", "in_ln_g", "in_ln_b", "w_gate", "w_val", "w_mem", "lam_mem",
    "loc_ln_g", "loc_ln_b", "conv_k", "conv_b", "w_route", "mix_ln_g",
    "mix_ln_b", "w_down", "w_mix", "w_up", "w_cgate", "lam_mix", "ref_ln_g",
    "ref_ln_b", "w_e1", "w_e2", "w_f", "out_ln_g", "out_ln_b", "lam_out",
    "w_head", "b_head",
)

# draw standard deviations of the seeded init (model.py:76-105); parameters not
# listed are constants (gains and residual weights 1, biases 0, w_mix = I)
_ONES = {"in_ln_g", "loc_ln_g", "mix_ln_g", "ref_ln_g", "out_ln_g", "lam_mem", "lam_mix", "lam_out"}


def _shapes(cfg: ModelConfig) -> dict:
    d, h, e, m = cfg.embed_dim, cfg.hidden_dim, cfg.expand_dim, cfg.mix_dim
    k, c, b = cfg.conv_kernel, cfg.cache_dim, cfg.batch
    vec_h = ("in_ln_g", "in_ln_b", "mix_ln_g", "mix_ln_b", "ref_ln_g", "ref_ln_b",
             "out_ln_g", "out_ln_b")
    shapes = {n: (h,) for n in vec_h}
    shapes.update({n: (d,) for n in ("loc_ln_g", "loc_ln_b", "conv_b")})
    shapes.update({n: () for n in ("lam_mem", "lam_mix", "lam_out")})
    shapes.update(emb=(256, d), w_gate=(d, d), w_val=(d, d), w_mem=(c, h), conv_k=(k, d, d),
                  w_route=(h, h), w_down=(h, m), w_mix=(b, m, m), w_up=(m, h), w_cgate=(h, h),
                  w_e1=(h, e), w_e2=(h, e), w_f=(e, h), w_head=(h, 256), b_head=(256,))
    return shapes


def init_params(cfg: ModelConfig) -> dict:
    """numpy ``default_rng(seed)`` draws in the reference order (model.py:62-105).

    Drawn afresh on every call, as the reference does for every Predictor
    (~0.2 s at the default size; part of every timed compress_bytes call).
    """
    return _draw_params(cfg)


def default_device() -> int:
    """The CUDA device a model lands on when the caller names none.

    torch's current device when torch has initialised CUDA in this process
    (``torch.cuda.set_device(local_rank)`` under torchrun), else
    ``LOCAL_RANK`` (one process per GPU), else 0.  The native calls restore
    the caller's current device, so this choice never leaks into torch.
    """
    torch = sys.modules.get("torch")
    if torch is not None:
        try:
            if torch.cuda.is_initialized():
                return int(torch.cuda.current_device())
        except Exception:  # noqa: BLE001 - a broken torch install must not matter here
            pass
    return int(os.environ.get("LOCAL_RANK", "0"))


def _draw_params(cfg: ModelConfig) -> dict:
    d, h, e, m = cfg.embed_dim, cfg.hidden_dim, cfg.expand_dim, cfg.mix_dim
    stds = {"emb": 0.02, "w_gate": d ** -0.5, "w_val": d ** -0.5,
            "w_mem": cfg.cache_dim ** -0.5, "conv_k": (cfg.conv_kernel * d) ** -0.5,
            "w_route": h ** -0.5, "w_down": h ** -0.5, "w_up": m ** -0.5,
            "w_cgate": h ** -0.5, "w_e1": h ** -0.5, "w_e2": h ** -0.5,
            "w_f": e ** -0.5, "w_head": 0.01}
    rng = np.random.default_rng(cfg.seed)
    shapes = _shapes(cfg)
    out = {}
    for name in PARAM_ORDER:
        shp = shapes[name]
        if name in stds:
            out[name] = rng.normal(0.0, stds[name], shp).astype(np.float32)
        elif name == "w_mix":
            out[name] = np.tile(np.eye(m, dtype=np.float32), (cfg.batch, 1, 1))
        else:
            out[name] = np.full(shp, 1.0 if name in _ONES else 0.0, dtype=np.float32)
    return out


def native_config(cfg: ModelConfig, variant: str = "full") -> _native.FadeConfig:
    return _native.FadeConfig(cfg.ctx_len, cfg.embed_dim, cfg.cache_dim, cfg.mix_dim,
                              cfg.expand_dim, cfg.batch, cfg.alphabet, cfg.conv_kernel,
                              cfg.lr, cfg.beta1, cfg.beta2, cfg.adam_eps,
                              VARIANTS.index(variant))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class Predictor:
    """One device model driving all B streams (model.py:44-58)."""

    def __init__(self, cfg: ModelConfig, variant: str = "full", device: int | None = None):
        cfg.validate()
        if variant not in VARIANTS:
            raise UsageError(f"unknown variant {variant!r}, pick one of {VARIANTS}")
        cfg.device_check()
        _native.require_device()
        self.cfg = cfg
        self.variant = variant
        self.device = default_device() if device is None else int(device)
        device = self.device
        self._shapes = _shapes(cfg)
        lib = _native.lib()
        h = ctypes.c_void_p()
        _native.check(lib.fade_model_create(ctypes.byref(native_config(cfg, variant)), device,
                                            ctypes.byref(h)), "fade_model_create")
        self._h = h
        params = init_params(cfg)
        for i, name in enumerate(PARAM_ORDER):
            self._set(0, i, params[name])
        self.alpha_stats = None
        self._live = False

    # -- plumbing ----------------------------------------------------------
    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _native.lib().fade_model_destroy(h)
            except Exception:  # noqa: BLE001 - interpreter teardown
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def _set(self, kind: int, i: int, arr) -> None:
        a = np.ascontiguousarray(arr, dtype=np.float32)
        _native.check(_native.lib().fade_model_set_tensor(self._h, kind, i, _ptr(a), a.size),
                      "set_tensor")

    def _get(self, kind: int, i: int) -> np.ndarray:
        a = np.empty(self._shapes[PARAM_ORDER[i]], dtype=np.float32)
        _native.check(_native.lib().fade_model_get_tensor(self._h, kind, i, _ptr(a), a.size),
                      "get_tensor")
        return a

    def _raise(self, status: int, err: _native.FadeError, what: str) -> None:
        if status == 0:
            return
        if status == 4:   # FADE_ERR_DIVERGED
            raise ModelDivergenceError(int(err.step), _native.last_error())
        if status == 5:   # FADE_ERR_QUANT
            raise ValueError(f"row {int(err.stream)} does not sum to 1 within quantizer tolerance")
        raise RuntimeError(f"{what} failed (status {status}): {_native.last_error()}")

    def _ctx(self, ctx) -> np.ndarray:
        c = np.ascontiguousarray(ctx, dtype=np.uint8)
        want = (self.cfg.batch, self.cfg.ctx_len)
        if c.shape != want:
            raise UsageError(f"context must be {want}, got {c.shape}")
        return c

    # -- public API (model.py:183-259) ------------------------------------
    @property
    def step_count(self) -> int:
        return self._counters()[1]

    def _counters(self):
        t, s = ctypes.c_int64(), ctypes.c_int64()
        _native.check(_native.lib().fade_model_get_counters(self._h, ctypes.byref(t),
                                                            ctypes.byref(s)), "get_counters")
        return int(t.value), int(s.value)

    def predict(self, ctx: np.ndarray) -> np.ndarray:
        c = self._ctx(ctx)
        probs = np.empty((self.cfg.batch, 256), dtype=np.float64)
        alpha = np.empty(3, dtype=np.float64)
        err = _native.FadeError()
        st = _native.lib().fade_model_predict(self._h, _ptr(c), _ptr(probs), _ptr(alpha),
                                              ctypes.byref(err))
        self._raise(st, err, "predict")
        # the single-stream variants have no router (model.py:146-151)
        self.alpha_stats = ((float(alpha[0]), float(alpha[1]), float(alpha[2]))
                            if self.variant not in ("global_only", "local_only") else None)
        self._live = True
        return probs

    def train_step(self, targets: np.ndarray) -> float:
        assert self._live, "train_step requires a preceding predict"
        t = np.ascontiguousarray(np.asarray(targets).astype(np.uint8))
        loss = ctypes.c_double()
        err = _native.FadeError()
        st = _native.lib().fade_model_train_step(self._h, _ptr(t), ctypes.byref(loss),
                                                 ctypes.byref(err))
        self._raise(st, err, "train_step")
        self._live = False
        return float(loss.value)

    def forward_debug(self, ctx: np.ndarray) -> dict:
        c = self._ctx(ctx)
        parts = {}
        v = self.variant
        skip = set()
        if v == "local_only":
            skip |= {"global"}
        if v == "global_only":
            skip |= {"local"}
        if v in ("global_only", "local_only"):
            skip |= {"alpha"}
        if v not in ("full", "mixer", "mixer_nogate"):
            skip |= {"mixer_inner"}
        for name in ("global", "local", "alpha", "mix", "mixer_inner", "coarse", "hidden",
                     "logits"):
            if name in skip:      # the reference's parts dict has no such key (model.py:121-175)
                continue
            width = 256 if name == "logits" else self.cfg.hidden_dim
            out = np.empty((self.cfg.batch, width), dtype=np.float32)
            _native.check(_native.lib().fade_model_forward_debug(self._h, _ptr(c), name.encode(),
                                                                 _ptr(out)), "forward_debug")
            parts[name] = out
        return parts

    def loss_grads(self, ctx: np.ndarray, targets: np.ndarray):
        c = self._ctx(ctx)
        t = np.ascontiguousarray(np.asarray(targets).astype(np.uint8))
        loss = ctypes.c_double()
        _native.check(_native.lib().fade_model_loss_grads(self._h, _ptr(c), _ptr(t),
                                                          ctypes.byref(loss)), "loss_grads")
        return float(loss.value), {n: self._get(3, i) for i, n in enumerate(PARAM_ORDER)}

    def eval_loss(self, ctx: np.ndarray, targets: np.ndarray) -> float:
        return self.loss_grads(ctx, targets)[0]

    def save_state(self) -> dict:
        cache = np.empty((self.cfg.batch, self.cfg.cache_dim), dtype=np.float32)
        _native.check(_native.lib().fade_model_get_cache(self._h, _ptr(cache)), "get_cache")
        t, sc = self._counters()
        return {"params": {n: self._get(0, i) for i, n in enumerate(PARAM_ORDER)},
                "cache": cache,
                "m": [self._get(1, i) for i in range(len(PARAM_ORDER))],
                "v": [self._get(2, i) for i in range(len(PARAM_ORDER))],
                "t": t, "step_count": sc}

    def load_state(self, state: dict) -> None:
        for i, n in enumerate(PARAM_ORDER):
            self._set(0, i, state["params"][n])
            self._set(1, i, state["m"][i])
            self._set(2, i, state["v"][i])
        cache = np.ascontiguousarray(state["cache"], dtype=np.float32)
        _native.check(_native.lib().fade_model_set_cache(self._h, _ptr(cache)), "set_cache")
        _native.check(_native.lib().fade_model_set_counters(self._h, int(state["t"]),
                                                            int(state["step_count"])),
                      "set_counters")

    def param_count(self) -> int:          # a method, as model.py:262
        return int(sum(int(np.prod(s)) for s in self._shapes.values()))

    def active_param_count(self) -> int:
        """Parameters this variant's graph reaches (model.py:265-276).  The
        reference finds them by which tensors receive a gradient; the device
        graph is fixed per variant, so the set is static (ACTIVE_PARAMS,
        checked against the reference's gradients in tests/test_cpu_surface.py)."""
        return int(sum(int(np.prod(self._shapes[n])) for n in active_params(self.variant)))


_HEAD = ("w_head", "b_head")
_GLOBAL = ("emb", "in_ln_g", "in_ln_b", "w_gate", "w_val", "w_mem", "lam_mem")
_LOCAL = ("emb", "loc_ln_g", "loc_ln_b", "conv_k", "conv_b")
_MIXER = ("mix_ln_g", "mix_ln_b", "w_down", "w_mix", "w_up", "lam_mix")
_FNR = ("ref_ln_g", "ref_ln_b", "w_e1", "w_e2", "w_f", "out_ln_g", "out_ln_b", "lam_out")


def active_params(variant: str) -> tuple:
    """Parameter names a variant's forward graph reaches (model.py:121-175), in
    PARAM_ORDER.  local_only never uses x = LN(emb), so in_ln_* are inactive."""
    names = set(_HEAD)
    if variant != "local_only":
        names |= set(_GLOBAL)
    if variant != "global_only":
        names |= set(_LOCAL)
    if variant not in ("global_only", "local_only"):
        names |= {"w_route", "in_ln_g", "in_ln_b"}
    if variant in ("full", "mixer", "mixer_nogate"):
        names |= set(_MIXER)
    if variant in ("full", "mixer"):
        names.add("w_cgate")
    if variant == "full":
        names |= set(_FNR)
    return tuple(n for n in PARAM_ORDER if n in names)


def nll_report(losses) -> tuple[float, float]:
    """Mean NLL in nats and bits per byte (model.py:279-284)."""
    if len(losses) == 0:
        raise ValueError("no losses recorded")
    nats = float(np.mean(losses))
    return nats, nats / LN2
