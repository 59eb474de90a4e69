"""A small compress -> decompress round trip for compute-sanitizer
(racecheck / synccheck / memcheck): the default-geometry kernels (B = 64 so
the run stays short), the three-stream PDL schedule, the CSPP coder stream
and the decoder in the head kernel, plus the Predictor API.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    from paper_2604_07239_b200 import ModelConfig, container, corpus
    from paper_2604_07239_b200.model import Predictor
    cfg = ModelConfig(batch=64, workers=1, seed=2)
    data = corpus.make_text(64 * 22, 3)          # 22 columns: 6 model steps
    blob, res = container.compress_bytes(data, cfg)
    assert container.decompress_bytes(blob) == data
    tiny = ModelConfig(ctx_len=4, embed_dim=8, cache_dim=32, mix_dim=8, expand_dim=32, batch=16,
                       workers=1, seed=1)
    m = Predictor(tiny)
    ctx = np.zeros((16, 4), np.uint8)
    m.predict(ctx)
    m.train_step(np.zeros(16, np.uint8))
    print("sanitize run ok", len(data), len(blob))


if __name__ == "__main__":
    main()
