"""TEST INFRASTRUCTURE ONLY: numpy restatement of the FADE predictor.

Forward (``pkg/src/dszip/model.py:109-179``, variant "full"), the explicit
backward that the reference's autograd graph evaluates (``nn/ops.py`` backward
closures, ``nn/tensor.py:37-58``), the float64 softmax / softmax-xent
(``nn/ops.py:246-279``) and bias-corrected Adam (``nn/optim.py:25-44``).

Arithmetic is float32 like the reference (``dtype=np.float64`` gives the fp64
twin used to bound the reference's own rounding noise). The B200 kernels are
checked against this file from transplanted state; this file is checked
against the reference's own outputs in tests/test_oracle.py.
"""

from __future__ import annotations

import math

import numpy as np

GELU_C = 0.7978845608   # ops.py:14
GELU_A = 0.044715       # ops.py:15
LN_EPS = 1e-5           # ops.py:16

# parameter order == Adam state order (model.py:76-105)
PARAM_ORDER = (
    "emb", "in_ln_g", "in_ln_b", "w_gate", "w_val", "w_mem", "lam_mem",
    "loc_ln_g", "loc_ln_b", "conv_k", "conv_b", "w_route", "mix_ln_g",
    "mix_ln_b", "w_down", "w_mix", "w_up", "w_cgate", "lam_mix", "ref_ln_g",
    "ref_ln_b", "w_e1", "w_e2", "w_f", "out_ln_g", "out_ln_b", "lam_out",
    "w_head", "b_head",
)


def param_shapes(cfg) -> dict:
    d, h, e, m = cfg.embed_dim, cfg.hidden_dim, cfg.expand_dim, cfg.mix_dim
    a, k, c, b = cfg.alphabet, cfg.conv_kernel, cfg.cache_dim, cfg.batch
    return {
        "emb": (a, d), "in_ln_g": (h,), "in_ln_b": (h,), "w_gate": (d, d),
        "w_val": (d, d), "w_mem": (c, h), "lam_mem": (), "loc_ln_g": (d,),
        "loc_ln_b": (d,), "conv_k": (k, d, d), "conv_b": (d,), "w_route": (h, h),
        "mix_ln_g": (h,), "mix_ln_b": (h,), "w_down": (h, m), "w_mix": (b, m, m),
        "w_up": (m, h), "w_cgate": (h, h), "lam_mix": (), "ref_ln_g": (h,),
        "ref_ln_b": (h,), "w_e1": (h, e), "w_e2": (h, e), "w_f": (e, h),
        "out_ln_g": (h,), "out_ln_b": (h,), "lam_out": (), "w_head": (h, a),
        "b_head": (a,),
    }


def init_params(cfg, dtype=np.float32) -> dict:
    """Seeded init in the reference's draw order (model.py:62-105)."""
    rng = np.random.default_rng(cfg.seed)
    d, h, e, m = cfg.embed_dim, cfg.hidden_dim, cfg.expand_dim, cfg.mix_dim
    shapes = param_shapes(cfg)
    std = {
        "emb": 0.02, "w_gate": d ** -0.5, "w_val": d ** -0.5,
        "w_mem": cfg.cache_dim ** -0.5, "conv_k": (cfg.conv_kernel * d) ** -0.5,
        "w_route": h ** -0.5, "w_down": h ** -0.5, "w_up": m ** -0.5,
        "w_cgate": h ** -0.5, "w_e1": h ** -0.5, "w_e2": h ** -0.5,
        "w_f": e ** -0.5, "w_head": 0.01,
    }
    ones = {"in_ln_g", "loc_ln_g", "mix_ln_g", "ref_ln_g", "out_ln_g",
            "lam_mem", "lam_mix", "lam_out"}
    p = {}
    for name in PARAM_ORDER:
        if name in std:   # draws happen in PARAM_ORDER, which is the reference order
            p[name] = rng.normal(0.0, std[name], shapes[name]).astype(dtype)
        elif name == "w_mix":
            p[name] = np.tile(np.eye(m, dtype=dtype), (cfg.batch, 1, 1))
        else:
            p[name] = np.full(shapes[name], 1.0 if name in ones else 0.0, dtype=dtype)
    return p


# -- elementwise pieces -----------------------------------------------------

def gelu(x):
    t = np.tanh(GELU_C * (x + GELU_A * x * x * x))
    return 0.5 * x * (1.0 + t)


def gelu_grad(x):
    t = np.tanh(GELU_C * (x + GELU_A * x * x * x))
    du = GELU_C * (1.0 + 3.0 * GELU_A * x * x)
    return 0.5 * (1.0 + t) + 0.5 * x * (1.0 - t * t) * du


def sigmoid(x):
    with np.errstate(over="ignore"):
        return 1.0 / (1.0 + np.exp(-x))


def ln_fwd(x, g, b):
    """Returns (out, xhat, inv) over the last axis (ops.py:94-101)."""
    mu = x.mean(axis=-1, keepdims=True)
    xc = x - mu
    var = (xc * xc).mean(axis=-1, keepdims=True)
    inv = 1.0 / np.sqrt(var + np.asarray(LN_EPS, dtype=x.dtype))
    xhat = xc * inv
    return xhat * g + b, xhat, inv


def ln_bwd(dy, xhat, inv, g):
    """Returns (dx, dgain, dbias) (ops.py:103-113)."""
    lead = tuple(range(dy.ndim - 1))
    db = dy.sum(axis=lead)
    dg = (dy * xhat).sum(axis=lead)
    gg = dy * g
    m1 = gg.mean(axis=-1, keepdims=True)
    m2 = (gg * xhat).mean(axis=-1, keepdims=True)
    return (gg - m1 - xhat * m2) * inv, dg, db


def softmax64(logits):
    z = logits.astype(np.float64)
    z = z - z.max(axis=-1, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=-1, keepdims=True)


def softmax_xent(logits, targets):
    """(mean nll nats, dlogits in logits dtype) -- ops.py:258-279."""
    z = logits.astype(np.float64)
    z = z - z.max(axis=-1, keepdims=True)
    logp = z - np.log(np.exp(z).sum(axis=-1, keepdims=True))
    rows = np.arange(targets.shape[0])
    loss = float(-logp[rows, targets].mean())
    d = np.exp(logp)
    d[rows, targets] -= 1.0
    d *= 1.0 / targets.shape[0]
    return loss, d.astype(logits.dtype)


# -- model --------------------------------------------------------------------

class OracleModel:
    """Single-context predictor with explicit backward; mirrors ``Predictor``."""

    def __init__(self, cfg, dtype=np.float32, params=None):
        self.cfg = cfg
        self.dtype = np.dtype(dtype)
        self.p = init_params(cfg, dtype) if params is None else {
            k: np.array(v, dtype=dtype) for k, v in params.items()}
        self.m = {k: np.zeros_like(v) for k, v in self.p.items()}
        self.v = {k: np.zeros_like(v) for k, v in self.p.items()}
        self.t = 0
        self.step_count = 0
        self.cache = np.zeros((cfg.batch, cfg.cache_dim), dtype=dtype)
        self._saved = None
        self.alpha_stats = None

    # state transfer, same dict shape as Predictor.save_state (model.py:239-259)
    def save_state(self) -> dict:
        return {"params": {k: v.copy() for k, v in self.p.items()},
                "cache": self.cache.copy(),
                "m": [self.m[k].copy() for k in PARAM_ORDER],
                "v": [self.v[k].copy() for k in PARAM_ORDER],
                "t": self.t, "step_count": self.step_count}

    def load_state(self, st: dict) -> None:
        for k, v in st["params"].items():
            self.p[k] = np.array(v, dtype=self.dtype)
        self.cache = np.array(st["cache"], dtype=self.dtype)
        for k, mm, vv in zip(PARAM_ORDER, st["m"], st["v"]):
            self.m[k] = np.array(mm, dtype=self.dtype)
            self.v[k] = np.array(vv, dtype=self.dtype)
        self.t = int(st["t"])
        self.step_count = int(st["step_count"])

    def forward(self, ctx):
        """Returns (logits, saved-activations); touches no state."""
        cfg, p = self.cfg, self.p
        bsz, d = cfg.batch, cfg.embed_dim
        ctx = np.asarray(ctx)
        s = {"ctx": ctx}
        emb = p["emb"][ctx]                                   # (B,T,D)
        x, s["x_hat"], s["x_inv"] = ln_fwd(emb.reshape(bsz, -1), p["in_ln_g"], p["in_ln_b"])
        s["x"] = x
        x_t = x[:, -d:]
        s["x_t"] = x_t
        s["gpre"] = x_t @ p["w_gate"]
        s["vpre"] = x_t @ p["w_val"]
        block = gelu(s["gpre"]) * s["vpre"]
        rolled = np.concatenate([self.cache[:, d:], block], axis=1)
        s["rolled"] = rolled
        s["upre"] = rolled @ p["w_mem"]
        h_g = gelu(s["upre"]) + x * p["lam_mem"]
        s["h_g"] = h_g
        loc, s["loc_hat"], s["loc_inv"] = ln_fwd(emb, p["loc_ln_g"], p["loc_ln_b"])
        k = cfg.conv_kernel
        pad = k // 2
        t = cfg.ctx_len
        xp = np.zeros((bsz, t + 2 * pad, d), dtype=self.dtype)
        xp[:, pad:pad + t] = loc
        s["loc_pad"] = xp
        conv = np.broadcast_to(p["conv_b"], (bsz, t, d)).copy()
        for j in range(k):
            conv += (xp[:, j:j + t].reshape(bsz * t, d) @ p["conv_k"][j]).reshape(bsz, t, d)
        s["conv"] = conv
        h_l = gelu(conv).reshape(bsz, -1)
        s["h_l"] = h_l
        s["rpre"] = x @ p["w_route"]
        alpha = sigmoid(s["rpre"])
        s["alpha"] = alpha
        h_mix = alpha * h_g + (1.0 - alpha) * h_l
        s["h_mix"] = h_mix
        z, s["z_hat"], s["z_inv"] = ln_fwd(h_mix, p["mix_ln_g"], p["mix_ln_b"])
        s["z"] = z
        s["zd"] = z @ p["w_down"]
        s["u"] = np.matmul(s["zd"][:, None, :], p["w_mix"])[:, 0, :]
        s["inner"] = s["u"] @ p["w_up"]
        s["cpre"] = h_mix @ p["w_cgate"]
        gate = sigmoid(s["cpre"])
        s["gate"] = gate
        h_c = s["inner"] * gate + h_mix * p["lam_mix"]
        s["h_c"] = h_c
        z2, s["z2_hat"], s["z2_inv"] = ln_fwd(h_c, p["ref_ln_g"], p["ref_ln_b"])
        s["z2"] = z2
        s["a1"] = z2 @ p["w_e1"]
        s["a2"] = z2 @ p["w_e2"]
        wide = gelu(s["a1"]) * s["a2"]
        s["wide"] = wide
        s["npre"] = wide @ p["w_f"]
        nrm, s["n_hat"], s["n_inv"] = ln_fwd(s["npre"], p["out_ln_g"], p["out_ln_b"])
        s["nrm"] = nrm
        h = gelu(nrm) + h_c * p["lam_out"]
        s["h"] = h
        logits = h @ p["w_head"] + p["b_head"]
        s["logits"] = logits
        return logits, s

    def backward(self, s, dl) -> dict:
        """Gradients of every parameter given dlogits (the autograd closures)."""
        cfg, p = self.cfg, self.p
        bsz, d, t = cfg.batch, cfg.embed_dim, cfg.ctx_len
        g = {}
        g["w_head"] = s["h"].T @ dl
        g["b_head"] = dl.sum(axis=0)
        dh = dl @ p["w_head"].T
        dh_c = dh * p["lam_out"]
        g["lam_out"] = np.asarray((dh * s["h_c"]).sum(), dtype=self.dtype)
        dn = dh * gelu_grad(s["nrm"])
        dnpre, g["out_ln_g"], g["out_ln_b"] = ln_bwd(dn, s["n_hat"], s["n_inv"], p["out_ln_g"])
        g["w_f"] = s["wide"].T @ dnpre
        dwide = dnpre @ p["w_f"].T
        da1 = dwide * s["a2"] * gelu_grad(s["a1"])
        da2 = dwide * gelu(s["a1"])
        g["w_e1"] = s["z2"].T @ da1
        g["w_e2"] = s["z2"].T @ da2
        dz2 = da1 @ p["w_e1"].T + da2 @ p["w_e2"].T
        dhc2, g["ref_ln_g"], g["ref_ln_b"] = ln_bwd(dz2, s["z2_hat"], s["z2_inv"], p["ref_ln_g"])
        dh_c = dh_c + dhc2
        dinner = dh_c * s["gate"]
        dcpre = dh_c * s["inner"] * s["gate"] * (1.0 - s["gate"])
        dh_mix = dh_c * p["lam_mix"]
        g["lam_mix"] = np.asarray((dh_c * s["h_mix"]).sum(), dtype=self.dtype)
        g["w_cgate"] = s["h_mix"].T @ dcpre
        dh_mix = dh_mix + dcpre @ p["w_cgate"].T
        g["w_up"] = s["u"].T @ dinner
        du = dinner @ p["w_up"].T
        g["w_mix"] = s["zd"][:, :, None] * du[:, None, :]
        dzd = np.matmul(du[:, None, :], p["w_mix"].transpose(0, 2, 1))[:, 0, :]
        g["w_down"] = s["z"].T @ dzd
        dz = dzd @ p["w_down"].T
        dhm2, g["mix_ln_g"], g["mix_ln_b"] = ln_bwd(dz, s["z_hat"], s["z_inv"], p["mix_ln_g"])
        dh_mix = dh_mix + dhm2
        alpha = s["alpha"]
        dalpha = dh_mix * (s["h_g"] - s["h_l"])
        dh_g = dh_mix * alpha
        dh_l = dh_mix * (1.0 - alpha)
        drpre = dalpha * alpha * (1.0 - alpha)
        g["w_route"] = s["x"].T @ drpre
        dx = drpre @ p["w_route"].T
        dupre = dh_g * gelu_grad(s["upre"])
        g["lam_mem"] = np.asarray((dh_g * s["x"]).sum(), dtype=self.dtype)
        dx = dx + dh_g * p["lam_mem"]
        g["w_mem"] = s["rolled"].T @ dupre
        dblock = dupre @ p["w_mem"][-d:, :].T       # roll_cache grads only the new block
        dgpre = dblock * s["vpre"] * gelu_grad(s["gpre"])
        dvpre = dblock * gelu(s["gpre"])
        g["w_gate"] = s["x_t"].T @ dgpre
        g["w_val"] = s["x_t"].T @ dvpre
        dx[:, -d:] += dgpre @ p["w_gate"].T + dvpre @ p["w_val"].T
        # local stream: gelu -> conv (taps ascending) -> LN_32
        dconv = dh_l.reshape(bsz, t, d) * gelu_grad(s["conv"])
        g["conv_b"] = dconv.sum(axis=(0, 1))
        k = cfg.conv_kernel
        pad = k // 2
        xp = s["loc_pad"]
        g2 = dconv.reshape(bsz * t, d)
        dk = np.empty_like(p["conv_k"])
        dxp = np.zeros_like(xp)
        for j in range(k):
            dk[j] = xp[:, j:j + t].reshape(bsz * t, d).T @ g2
            dxp[:, j:j + t] += (g2 @ p["conv_k"][j].T).reshape(bsz, t, d)
        g["conv_k"] = dk
        demb, g["loc_ln_g"], g["loc_ln_b"] = ln_bwd(dxp[:, pad:pad + t], s["loc_hat"],
                                                    s["loc_inv"], p["loc_ln_g"])
        dxf, g["in_ln_g"], g["in_ln_b"] = ln_bwd(dx, s["x_hat"], s["x_inv"], p["in_ln_g"])
        demb = demb + dxf.reshape(bsz, t, d)
        de = np.zeros_like(p["emb"])
        np.add.at(de, s["ctx"].reshape(-1), demb.reshape(-1, d))
        g["emb"] = de
        return g

    def adam(self, grads) -> None:
        """optim.py:25-44, including the float64 bias-correction multiply."""
        cfg = self.cfg
        self.t += 1
        c1 = 1.0 - cfg.beta1 ** self.t
        c2 = 1.0 - cfg.beta2 ** self.t
        step = cfg.lr / c1
        inv_sqrt_c2 = 1.0 / np.sqrt(c2)
        for name in PARAM_ORDER:
            gr = grads[name]
            m, v, w = self.m[name], self.v[name], self.p[name]
            m *= cfg.beta1
            m += (1.0 - cfg.beta1) * gr
            v *= cfg.beta2
            v += (1.0 - cfg.beta2) * (gr * gr)
            sc = np.empty_like(v)
            np.sqrt(v, out=sc)
            sc *= inv_sqrt_c2
            sc += cfg.adam_eps
            np.divide(m, sc, out=sc)
            sc *= step
            w -= sc

    # -- Predictor-like surface --------------------------------------------
    def predict(self, ctx):
        logits, s = self.forward(ctx)
        if not np.all(np.isfinite(logits)):
            raise FloatingPointError(f"non-finite logits at step {self.step_count}")
        self.cache = s["rolled"]
        a = s["alpha"]
        self.alpha_stats = (float(a.mean()), float(a.min()), float(a.max()))
        self._saved = s
        return softmax64(logits)

    def train_step(self, targets) -> float:
        s = self._saved
        assert s is not None, "train_step requires a preceding predict"
        loss, dl = softmax_xent(s["logits"], np.asarray(targets, dtype=np.int64))
        if not math.isfinite(loss):
            raise FloatingPointError(f"non-finite loss at step {self.step_count}")
        self.adam(self.backward(s, dl))
        self._saved = None
        self.step_count += 1
        return loss

    def loss_grads(self, ctx, targets):
        logits, s = self.forward(ctx)
        loss, dl = softmax_xent(logits, np.asarray(targets, dtype=np.int64))
        return loss, self.backward(s, dl)
