"""Container size + sha of the criterion-5 workload (1 MiB text, seed 5) with
whatever library FADE_LIB_PATH selects: cross-process / cross-build
determinism check."""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_07239_b200 import ModelConfig, container, corpus  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
data = corpus.make_text(n, 12)
blob, res = container.compress_bytes(data, ModelConfig(seed=5))
print(len(blob), hashlib.sha256(blob[98:]).hexdigest()[:16], repr(res.losses[-1]))
