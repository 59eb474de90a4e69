"""One-step probability error of the device model against the reference's
goldens (tiny, mid: transplanted state; default: 3 steps from the seeded
init), as max-abs and mean KL in bits/symbol.

    python tools/kl_check.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def kl_bits(p, q):
    return float(np.mean(np.sum(p * (np.log2(p) - np.log2(q)), axis=1)))


def main():
    from conftest import load_golden, model_golden
    from paper_2604_07239_b200 import ModelConfig, corpus
    from paper_2604_07239_b200.model import Predictor
    from paper_2604_07239_b200.pipeline import StreamPartition
    out = {}
    for name in ("tiny", "mid"):
        cfg, st, z = model_golden(name)
        m = Predictor(cfg)
        m.load_state(st)
        p = m.predict(z["ctx"])
        ref = z["next_probs"]
        out[name] = {"max_abs": float(np.abs(p - ref).max()), "kl_bits": kl_bits(ref, p)}
    z = load_golden("model_default_digest.npz")
    cfg = ModelConfig(seed=5)
    data = corpus.make_text(1 << 20, 12)
    mat = StreamPartition.from_length(len(data), cfg.batch).split(data)
    m = Predictor(cfg)
    t = cfg.ctx_len
    for j in range(z["probs"].shape[0]):
        i = t + j
        p = m.predict(mat[:, i - t:i])[:z["probs"].shape[1]]
        ref = z["probs"][j]
        out[f"default_step{j}"] = {"max_abs": float(np.abs(p - ref).max()), "kl_bits": kl_bits(ref, p)}
        m.train_step(mat[:, i])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
