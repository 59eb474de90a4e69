"""Large-size bits/byte oracle (test infrastructure): runs oracle/torch_model.py
(fp32 PyTorch-eager restatement of the reference's online loop, TF32 off) over
a workload exactly as run_serial_compress sequences it (StreamPartition, warm-up
columns uniform-coded, predict -> code -> train per column) and estimates the
reference's container size from the model's own float64 probabilities:

    bytes ~= sum(-log2 (freq[symbol] / 65536)) / 8 over the model steps
             + warm * B (uniform warm-up: exactly 1 byte per symbol)
             + 4 * B (coder tails) + 98 + 8 * B (header)

where freq is the reference's quantiser (kernels.py:87-113, vectorised here in
torch: floor, largest remainders by the same int64 keys, zero raise from the
first maximum) applied to the oracle's float64 probabilities, so the estimate
carries the quantiser's 16-bit floor (large for low-entropy data such as DNA).
Checked against the reference's real container at the criterion-5 workload
(1 MiB text, 233,320 B).  Prints one JSON line per workload; with --gpu also
compresses the same bytes with this package (compress_bytes, lossless check)
so the two can be compared at sizes the CPU reference cannot finish.

    python tools/bpb_oracle.py text:1048576:12 dna:4194304:3 --gpu
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


KEYSCALE = float(1 << 40)   # kernels.py _KEYSCALE


def quantize_t(p):
    """kernels.py:87-113 (_np_quantize_rows) on a float64 [R,256] torch tensor."""
    import torch
    a = p.shape[1]
    t = p * 65536.0
    v = t.to(torch.int64)
    deficit = 65536 - v.sum(dim=1)
    frac = t - v.double()
    keys = (frac * KEYSCALE).to(torch.int64) * 256 + (a - 1 - torch.arange(a, device=p.device))
    order = torch.argsort(keys, dim=1)
    rank = torch.empty_like(order)
    rank.scatter_(1, order, torch.arange(a, device=p.device).expand_as(order).contiguous())
    v = v + (rank >= (a - deficit)[:, None]).to(torch.int64)
    zeros = (v == 0).sum(dim=1)
    imax = v.argmax(dim=1)
    rows = torch.arange(v.shape[0], device=p.device)
    v[rows, imax] = v[rows, imax] - zeros
    return torch.clamp(v, min=1)


def oracle_run(data, cfg, tf32=False):
    import numpy as np
    import torch
    from oracle.torch_model import TorchOracle
    from paper_2604_07239_b200.pipeline import StreamPartition
    part = StreamPartition.from_length(len(data), cfg.batch)
    mat = part.split(data)
    L = part.stream_length
    T = cfg.ctx_len
    warm = min(T, L)
    dmat = torch.from_numpy(np.ascontiguousarray(mat)).cuda().long()
    m = TorchOracle(cfg, tf32=tf32)
    bits = torch.zeros((), dtype=torch.float64, device="cuda")
    qbits = torch.zeros((), dtype=torch.float64, device="cuda")
    losses = torch.zeros(max(L - warm, 1), dtype=torch.float64, device="cuda")
    for i in range(warm, L):
        p = m.predict(dmat[:, i - T:i], check=False)
        y = dmat[:, i]
        bits += -torch.log2(p.gather(1, y[:, None])).sum()
        f = quantize_t(p).gather(1, y[:, None]).double()
        qbits += -torch.log2(f / 65536.0).sum()
        losses[i - warm] = m.train_step_t(y)
    if not bool(torch.isfinite(bits)):
        raise FloatingPointError("oracle diverged")
    B = cfg.batch
    fixed = warm * B + 4 * B + 98 + 8 * B
    est = math.ceil(float(qbits) / 8.0) + fixed
    ideal = math.ceil(float(bits) / 8.0) + fixed
    return est, ideal, float(losses[:L - warm].mean()) if L > warm else 0.0, L - warm


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workloads", nargs="+", help="kind:n:seed")
    ap.add_argument("--gpu", action="store_true", help="also compress with this package")
    ap.add_argument("--tf32", action="store_true",
                    help="diagnostic: the oracle's GEMMs on TF32 tensor cores instead of fp32")
    a = ap.parse_args()
    from paper_2604_07239_b200 import ModelConfig, container, corpus
    for spec in a.workloads:
        kind, n, seed = spec.split(":")
        data = getattr(corpus, "make_" + kind)(int(n), int(seed))
        cfg = ModelConfig(seed=5).shrink_to_fit(len(data))
        t0 = time.perf_counter()
        est, ideal, mean_loss, steps = oracle_run(data, cfg, a.tf32)
        rec = {"workload": f"make_{kind}({n}, {seed}), ModelConfig(seed=5)", "steps": steps,
               "oracle_gemms": "tf32" if a.tf32 else "fp32",
               "oracle_bytes_est": est, "oracle_bpb_est": 8.0 * est / len(data),
               "oracle_bytes_unquantised": ideal,
               "oracle_mean_loss_nats": mean_loss, "oracle_s": time.perf_counter() - t0}
        if a.gpu:
            t0 = time.perf_counter()
            blob, res = container.compress_bytes(data, ModelConfig(seed=5))
            rec.update(gpu_bytes=len(blob), gpu_bpb=8.0 * len(blob) / len(data),
                       gpu_mean_loss_nats=float(sum(res.losses) / max(1, len(res.losses))),
                       gpu_compress_s=time.perf_counter() - t0,
                       lossless=container.decompress_bytes(blob) == data,
                       rel_gap_vs_oracle=len(blob) / est - 1.0)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
