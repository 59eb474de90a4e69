"""Bits/byte parity evidence (acceptance criterion 5 workload): default config
(seed 5), make_text(1 MiB, 12), pipelined compress -> container -> decompress.
Prints one JSON line with sizes, bits/byte, the reference's size (BASELINE.md
section 2: 233,320 B = 1.7801 bpb), the relative gap, timings and the
round-trip check.  Extra workloads can be named with --extra (n:seed:kind)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--extra", default="")
    ap.add_argument("--only-extra", action="store_true", help="skip the 1 MiB reference case")
    a = ap.parse_args()
    from paper_2604_07239_b200 import ModelConfig, container, corpus
    cases = [] if a.only_extra else [(1 << 20, 12, "text", 233320)]
    for spec in filter(None, a.extra.split(",")):
        n, seed, kind = spec.split(":")
        cases.append((int(n), int(seed), kind, None))
    for n, seed, kind, ref in cases:
        data = getattr(corpus, "make_" + kind)(n, seed)
        cfg = ModelConfig(seed=5)
        t0 = time.perf_counter()
        blob, res = container.compress_bytes(data, cfg)
        tc = time.perf_counter() - t0
        t0 = time.perf_counter()
        back = container.decompress_bytes(blob)
        td = time.perf_counter() - t0
        line = {"workload": f"make_{kind}({n}, {seed}), ModelConfig(seed=5)", "bytes": len(blob),
                "compress_MBps": n / tc / 1e6, "decompress_MBps": n / td / 1e6,
                "bits_per_byte": 8.0 * len(blob) / n, "lossless": back == data,
                "compress_s": tc, "decompress_s": td, "mean_loss_nats": sum(res.losses) / len(res.losses)}
        if ref:
            line.update(reference_bytes=ref, reference_bpb=8.0 * ref / n,
                        rel_gap=(len(blob) - ref) / ref)
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
