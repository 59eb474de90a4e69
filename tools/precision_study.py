"""TF32 operand-rounding study: KL of one-step
probabilities against the reference's own (tests/golden model_<cfg>.npz,
next_probs from transplanted state) when the tensor-core GEMMs of the forward
round their operands differently.  CPU only (numpy emulation of
tcgen05.mma.kind::tf32, which truncates fp32 operands to a 10-bit mantissa;
the 32x32 gate/value GEMMs, the conv and the per-stream W_U product run in
fp32 on CUDA cores on the B200 and stay fp32 here).

    python tools/precision_study.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

TC_WEIGHTS = ("w_mem", "w_route", "w_down", "w_up", "w_cgate", "w_e1", "w_e2", "w_f", "w_head")


def tf32(a, mode):
    a = np.ascontiguousarray(a, dtype=np.float32)
    if mode == "fp32":
        return a
    u = a.view(np.uint32).astype(np.uint64)
    if mode == "rne":
        u = u + 0xFFF + ((u >> 13) & 1)
    return (u & 0xFFFFE000).astype(np.uint32).view(np.float32)


def split3(a):
    """3xTF32 operand split: hi = tf32(a), lo = tf32(a - hi)."""
    hi = tf32(a, "trunc")
    return hi, tf32(np.asarray(a, np.float32) - hi, "trunc")


class W(np.ndarray):
    """A weight whose `x @ W` runs like a tensor-core GEMM: activation
    operand rounded with `amode`, weight with `wmode` ('3x' = 3xTF32).
    `per` maps a weight name to its own activation mode (overrides amode)."""
    amode = "trunc"
    wmode = "trunc"
    per = {}

    def __rmatmul__(self, other):
        a, w = np.asarray(other, np.float32), np.asarray(self, np.float32)
        am = W.per.get(getattr(self, "wname", ""), W.amode)
        if am == "3x":
            ah, al = split3(a)
            wh, wl = split3(w)
            return np.matmul(ah, wh) + (np.matmul(ah, wl) + np.matmul(al, wh))
        return np.matmul(tf32(a, am), tf32(w, W.wmode))


def kl_bits(ref, p):
    return float(np.mean(np.sum(ref * (np.log2(ref) - np.log2(p)), axis=1)))


def main():
    from conftest import model_golden
    from oracle.model import OracleModel, softmax64
    modes = {"fp32": ("fp32", "fp32"), "trunc (tcgen05 today)": ("trunc", "trunc"),
             "activations RNE, weights trunc": ("rne", "trunc"),
             "activations trunc, weights RNE": ("trunc", "rne"), "both RNE": ("rne", "rne"),
             "3xTF32": ("3x", "3x"),
             # RNE at the producing kernel for the operands that are only ever
             # GEMM inputs (cache, z, u, z2, wide, h); x and h_mix also feed
             # fp32 residuals and stay truncated by the MMA
             "GEMM-only activations RNE at source": ("sel", "trunc")}
    sel = {"w_mem": "rne", "w_route": "trunc", "w_down": "rne", "w_up": "rne",
           "w_cgate": "trunc", "w_e1": "rne", "w_e2": "rne", "w_f": "rne", "w_head": "rne"}
    out = {}
    for name in ("tiny", "mid"):
        cfg, st, z = model_golden(name)
        ref = z["next_probs"]
        for label, (am, wm) in modes.items():
            m = OracleModel(cfg)
            m.load_state(st)
            W.amode, W.wmode = (am if am != "sel" else "trunc"), wm
            W.per = sel if am == "sel" else {}
            for k in TC_WEIGHTS:
                m.p[k] = m.p[k].view(W)
                m.p[k].wname = k
            lg, _ = m.forward(z["ctx"])
            p = softmax64(np.asarray(lg))
            out.setdefault(name, {})[label] = {"max_abs": float(np.abs(p - ref).max()),
                                               "kl_bits": kl_bits(ref, p)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
