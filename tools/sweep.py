"""B sweep on one B200 (BASELINE.json config 3): compress MB/s and timestep
time for B = 64 ... 4096 at default dims, device-resident 100 MB text,
graph-replayed timesteps (same method as bench.py's `value`).

    python tools/sweep.py [--batches 64,128,...] [--steps 256]
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", default="64,128,256,512,1024,2048,4096")
    ap.add_argument("--steps", type=int, default=256)
    ap.add_argument("--size", type=int, default=100_000_000)
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_2604_07239_b200 import ModelConfig, _native, corpus
    from paper_2604_07239_b200.model import Predictor
    from paper_2604_07239_b200.pipeline import StreamPartition
    lib = _native.lib()
    data = corpus.make_text(a.size, 12)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650, "bf16_tflops": 1590}
    for b in [int(x) for x in a.batches.split(",")]:
        cfg = ModelConfig(batch=b, workers=1)
        part = StreamPartition.from_length(len(data), b)
        mat = torch.from_numpy(np.ascontiguousarray(part.split(data))).cuda()
        m = Predictor(cfg)
        sp = ctypes.c_void_p()
        lib.fade_model_stream(m.handle, ctypes.byref(sp))
        stream = torch.cuda.ExternalStream(sp.value)
        coder, la = ctypes.c_void_p(), ctypes.c_int()
        run = lambda n: _native.check(lib.fade_bench_compress_steps(
            m.handle, mat.data_ptr(), part.stream_length, cfg.ctx_len, n, ctypes.byref(coder),
            ctypes.byref(la), None), "steps")
        run(8)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run(a.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        P = 15_484_259 + 16_384 * b
        t_roof = max(24.0 * P / (peaks["hbm_gbs"] * 1e9), 2.0 * b * 44_521_472 / (peaks["bf16_tflops"] / 2 * 1e12))
        print(json.dumps({"batch": b, "ms_per_timestep": ms, "MBps": b / ms / 1e3,
                          "roofline_MBps": b / t_roof / 1e6, "frac": t_roof * 1e3 / ms}), flush=True)
        lib.fade_coder_destroy(coder)
        del m, mat
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
