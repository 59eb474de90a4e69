"""Time the dominant step components alone (fade_bench_probe) at several B:
the FNR expand GEMM, the W12 update, the W_route/W_mem update, the W_U
update (bmm_bwd), the FNR project GEMM and the trunk / small-parameter
kernels, each `iters` back-to-back
launches on the model stream after a few real timesteps.

    python tools/probe.py [--batches 512,4096] [--iters 20]
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NAMES = {0: "e12", 1: "w12_update", 2: "wroute_wmem_update", 3: "bmm_bwd", 4: "f_project",
         5: "trunk_bwd", 6: "trunk_fwd", 7: "small_adam"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", default="512,4096")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--which", default="", help="comma list of component names (default all)")
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_2604_07239_b200 import ModelConfig, _native, corpus
    from paper_2604_07239_b200.model import Predictor
    from paper_2604_07239_b200.pipeline import StreamPartition
    lib = _native.lib()
    for b in [int(x) for x in a.batches.split(",")]:
        cfg = ModelConfig(batch=b, workers=1)
        data = corpus.make_text(b * 64, 12)
        part = StreamPartition.from_length(len(data), b)
        mat = torch.from_numpy(np.ascontiguousarray(part.split(data))).cuda()
        m = Predictor(cfg)
        coder, la = ctypes.c_void_p(), ctypes.c_int()
        _native.check(lib.fade_bench_compress_steps(m.handle, mat.data_ptr(), part.stream_length,
                                                    cfg.ctx_len, 4, ctypes.byref(coder),
                                                    ctypes.byref(la), None), "steps")
        torch.cuda.synchronize()
        out = {"batch": b}
        for w, name in NAMES.items():
            if a.which and name not in a.which.split(","):
                continue
            ms, by, fl = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
            _native.check(lib.fade_bench_probe(m.handle, w, a.iters, ctypes.byref(ms),
                                               ctypes.byref(by), ctypes.byref(fl)), "probe")
            out[name] = {"us": round(ms.value * 1e3, 2), "GB/s": round(by.value / ms.value / 1e6),
                         "TF/s": round(fl.value / ms.value / 1e9)} if by.value else \
                {"us": round(ms.value * 1e3, 2)}
        print(json.dumps(out), flush=True)
        lib.fade_coder_destroy(coder)
        del m, mat
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
