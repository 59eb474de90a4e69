"""Per-CTA phase timing of the two largest GEMMs inside a real timestep.

`make probe` builds build/probe/libfade_b200.so with -DFADE_PHASE_PROBE: the
W12 weight-update GEMM (k_gemm_tf32<256,0,2,2>, one tile per CTA) stamps
%globaltimer after its PDL wait, when its accumulator is complete and when its
last Adam chunk is stored; the persistent e12 GEMM (k_gemm_ws<256,2>) stamps
its start, each accumulator hand-over and its end.  This script runs 3 graph
timesteps, then each GEMM alone, and prints the phase distribution over CTAs.

    make probe && FADE_LIB_PATH=build/probe/libfade_b200.so python tools/phase_probe.py
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from paper_2604_07239_b200 import ModelConfig, _native, corpus
    from paper_2604_07239_b200.model import Predictor
    from paper_2604_07239_b200.pipeline import StreamPartition
    lib = _native.lib()
    if not hasattr(lib, "fade_debug_phase"):
        sys.exit("not a probe build: make probe; FADE_LIB_PATH=build/probe/libfade_b200.so")
    cfg = ModelConfig(batch=512, workers=1)
    data = corpus.make_text(4_000_000, 12)
    part = StreamPartition.from_length(len(data), cfg.batch)
    dmat = torch.from_numpy(np.ascontiguousarray(part.split(data))).cuda()
    m = Predictor(cfg)

    def table():
        torch.cuda.synchronize()
        a = np.zeros((2048, 4), np.uint64)
        assert lib.fade_debug_phase(a.ctypes.data_as(ctypes.c_void_p)) == 0
        return a.astype(np.int64)

    def stats(name, rows, cols):
        t0 = rows[:, 0][rows[:, 0] > 0].min()
        print(f"  {name}: span {(rows[:, cols[-1][1]].max() - t0) / 1e3:.1f} us over {len(rows)} CTAs")
        for label, j in cols:
            c = rows[:, j][rows[:, j] > 0]
            c = (c - t0) / 1e3
            print(f"    {label:18s} n={len(c):3d} min {c.min():6.1f} med {np.median(c):6.1f} max {c.max():6.1f} us")

    def report(tag):
        a = table()
        print(f"== {tag}")
        stats("W12 update (one tile per CTA)", a[:256],
              [("start", 0), ("accumulator done", 1), ("Adam chunks done", 2)])
        stats("e12 (persistent)", a[1024:1024 + 148],
              [("start", 0), ("tile 1 accum", 1), ("tile 2 accum", 2), ("end", 3)])

    coder, la = ctypes.c_void_p(), ctypes.c_int()
    _native.check(lib.fade_bench_compress_steps(m.handle, dmat.data_ptr(), part.stream_length, 16, 3,
                                                ctypes.byref(coder), ctypes.byref(la), None), "steps")
    report("inside the timestep graph")
    ms, by, fl = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    for which in (1, 0):
        _native.check(lib.fade_bench_probe(m.handle, which, 20, ctypes.byref(ms), ctypes.byref(by),
                                           ctypes.byref(fl)), "probe")
    report("each GEMM alone (fade_bench_probe)")


if __name__ == "__main__":
    main()
