"""The bench hook's captured timestep belongs to its model: a model created at
the address of a destroyed one (the allocator reuses it) must not replay the
old model's graph (tools/sweep.py hit an illegal address that way at B=2048)."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_bench_graph_not_reused_across_models():
    import torch
    from paper_2604_07239_b200 import ModelConfig, _native, corpus
    from paper_2604_07239_b200.model import Predictor
    from paper_2604_07239_b200.pipeline import StreamPartition
    lib = _native.lib()
    data = corpus.make_text(200_000, 3)
    for b in (64, 128, 64, 256):
        cfg = ModelConfig(batch=b, workers=1)
        part = StreamPartition.from_length(len(data), b)
        mat = torch.from_numpy(np.ascontiguousarray(part.split(data))).cuda()
        m = Predictor(cfg)
        coder, la = ctypes.c_void_p(), ctypes.c_int()
        _native.check(lib.fade_bench_compress_steps(m.handle, mat.data_ptr(), part.stream_length,
                                                    cfg.ctx_len, 4, ctypes.byref(coder),
                                                    ctypes.byref(la), None), "steps")
        torch.cuda.synchronize()
        assert la.value > 0
        lib.fade_coder_destroy(coder)
        del m, mat
