"""TEST INFRASTRUCTURE ONLY: an fp32 PyTorch-eager restatement of the FADE
predictor's online loop, the large-size bits/byte oracle (SURVEY.md section
8d: "optionally a test-only PyTorch-eager fp32 restatement of model.py as a
secondary large-size bpb oracle, validated first against the CPU at 1 MiB").

The CPU reference needs ~0.3-0.6 s per timestep, so it cannot code 4 MiB or
100 MB; this restatement runs the same arithmetic -- fp32 GEMMs with TF32
disabled, float64 softmax / softmax-xent, bias-corrected Adam in the
reference's order (``pkg/src/dszip/model.py:109-215``, ``nn/ops.py``,
``nn/optim.py:25-44``; forward as oracle/model.py) -- on a GPU with autograd,
at a few ms per timestep.  It is never imported by the product package; only
tools/bpb_oracle.py and tests use it.
"""

from __future__ import annotations

import math

import numpy as np

from .model import PARAM_ORDER, init_params

GELU_C = 0.7978845608   # ops.py:14
GELU_A = 0.044715       # ops.py:15
LN_EPS = 1e-5           # ops.py:16


class TorchOracle:
    """Predictor.predict / train_step (model.py:183-215) on torch tensors."""

    def __init__(self, cfg, device="cuda", tf32=False):
        import torch
        # tf32=True is a diagnostic only: cuBLAS TF32 GEMMs (operands rounded
        # to a 10-bit mantissa), to separate precision effects on long runs
        torch.backends.cuda.matmul.allow_tf32 = tf32
        torch.backends.cudnn.allow_tf32 = tf32
        self.torch = torch
        self.cfg = cfg
        self.dev = device
        host = init_params(cfg)
        self.p = {k: torch.tensor(np.asarray(v), device=device).requires_grad_(True)
                  for k, v in host.items()}
        self.m = {k: torch.zeros_like(v) for k, v in self.p.items()}
        self.v = {k: torch.zeros_like(v) for k, v in self.p.items()}
        self.cache = torch.zeros(cfg.batch, cfg.cache_dim, device=device)
        self.t = 0
        self._live = None

    def _ln(self, x, g, b):
        mu = x.mean(dim=-1, keepdim=True)
        c = x - mu
        var = (c * c).mean(dim=-1, keepdim=True)
        return c / self.torch.sqrt(var + LN_EPS) * g + b

    @staticmethod
    def _gelu(x, torch):
        return 0.5 * x * (1.0 + torch.tanh(GELU_C * (x + GELU_A * x * x * x)))

    def forward(self, ctx):
        torch, p, cfg = self.torch, self.p, self.cfg
        bsz, d, t = cfg.batch, cfg.embed_dim, cfg.ctx_len
        gelu = lambda x: self._gelu(x, torch)
        emb = p["emb"][ctx]                                         # (B,T,D)
        x = self._ln(emb.reshape(bsz, -1), p["in_ln_g"], p["in_ln_b"])
        x_t = x[:, -d:]
        block = gelu(x_t @ p["w_gate"]) * (x_t @ p["w_val"])
        rolled = torch.cat([self.cache[:, d:], block], dim=1)       # old cache detached
        h_g = gelu(rolled @ p["w_mem"]) + x * p["lam_mem"]
        loc = self._ln(emb, p["loc_ln_g"], p["loc_ln_b"])
        k = cfg.conv_kernel
        xp = torch.nn.functional.pad(loc, (0, 0, k // 2, k // 2))
        conv = p["conv_b"].expand(bsz, t, d)
        for j in range(k):                                          # taps ascending (ops.py:70-72)
            conv = conv + xp[:, j:j + t] @ p["conv_k"][j]
        h_l = gelu(conv).reshape(bsz, -1)
        alpha = torch.sigmoid(x @ p["w_route"])
        h_mix = alpha * h_g + (1.0 - alpha) * h_l
        z = self._ln(h_mix, p["mix_ln_g"], p["mix_ln_b"])
        u = torch.bmm((z @ p["w_down"])[:, None, :], p["w_mix"])[:, 0, :]
        h_c = (u @ p["w_up"]) * torch.sigmoid(h_mix @ p["w_cgate"]) + h_mix * p["lam_mix"]
        z2 = self._ln(h_c, p["ref_ln_g"], p["ref_ln_b"])
        wide = gelu(z2 @ p["w_e1"]) * (z2 @ p["w_e2"])
        nrm = self._ln(wide @ p["w_f"], p["out_ln_g"], p["out_ln_b"])
        h = gelu(nrm) + h_c * p["lam_out"]
        return h @ p["w_head"] + p["b_head"], rolled.detach()

    def _idx(self, a):
        torch = self.torch
        if isinstance(a, torch.Tensor):
            return a.to(self.dev).long()
        return torch.as_tensor(np.asarray(a, np.int64), device=self.dev)

    def predict(self, ctx, check=True):
        """float64 probabilities (ops.py:246-255); commits the rolled cache.
        check=False skips the host-side finite check (no device sync)."""
        torch = self.torch
        logits, rolled = self.forward(self._idx(ctx))
        if check and not bool(torch.isfinite(logits).all()):
            raise FloatingPointError("non-finite logits")
        self.cache = rolled
        self._live = logits
        return torch.softmax(logits.detach().double(), dim=-1)

    def train_step(self, targets):
        return float(self.train_step_t(targets))

    def train_step_t(self, targets):
        """softmax-xent in float64 (ops.py:258-279), backward, Adam (optim.py:25-44);
        returns the loss as a device scalar (no sync)."""
        torch, cfg = self.torch, self.cfg
        tg = self._idx(targets)
        lg = self._live
        self._live = None
        lp = torch.log_softmax(lg.detach().double(), dim=-1)
        loss = -lp.gather(1, tg[:, None]).mean()
        # d loss / d logits = (p - onehot) / B, computed in f64 and cast to f32
        grad = (torch.exp(lp) - torch.nn.functional.one_hot(tg, lg.shape[1]).double()) / lg.shape[0]
        lg.backward(grad.float())
        self.t += 1
        c1 = 1.0 - cfg.beta1 ** self.t
        c2 = 1.0 - cfg.beta2 ** self.t
        step, inv_sqrt_c2 = cfg.lr / c1, 1.0 / math.sqrt(c2)
        with torch.no_grad():
            for name in PARAM_ORDER:
                w = self.p[name]
                g = w.grad
                m, v = self.m[name], self.v[name]
                m.mul_(cfg.beta1).add_((1.0 - cfg.beta1) * g)
                v.mul_(cfg.beta2).add_((1.0 - cfg.beta2) * (g * g))
                sc = (torch.sqrt(v).double() * inv_sqrt_c2).float() + cfg.adam_eps
                w.sub_(m / sc * step)
                w.grad = None
        return loss
