"""Reference-side bits/byte at workloads beyond criterion 5:
runs the reference's own compress_bytes (dszip, installed unmodified into
baseline/_ref, or importable from /root/reference/pkg/src) on 1 MiB DNA and
mixed inputs from this package's corpus generators (byte-identical to the
reference's _corpus, tests/golden/corpus_digest.json) at the default config,
seed 5.  Each run takes ~20 min on 8 cores (2,048 online steps); writes one
JSON line per workload to stdout.

    python tests/golden/make_bpb_ref.py dna:1048576:3 >> tests/golden/bpb_ref.jsonl
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(p):
        sys.path.insert(0, p)
        break


def main():
    from dszip.config import ModelConfig
    from dszip.container import compress_bytes
    from paper_2604_07239_b200 import corpus
    for spec in sys.argv[1:]:
        kind, n, seed = spec.split(":")
        data = getattr(corpus, "make_" + kind)(int(n), int(seed))
        t0 = time.perf_counter()
        blob, res = compress_bytes(data, ModelConfig(seed=5))
        print(json.dumps({"workload": f"make_{kind}({n}, {seed}), ModelConfig(seed=5)",
                          "kind": kind, "n": int(n), "seed": int(seed), "bytes": len(blob),
                          "bits_per_byte": 8.0 * len(blob) / len(data),
                          "mean_loss_nats": float(sum(res.losses) / max(1, len(res.losses))),
                          "seconds": time.perf_counter() - t0}), flush=True)


if __name__ == "__main__":
    main()
