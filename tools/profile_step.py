import ctypes, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2604_07239_b200 import ModelConfig, _native, corpus
from paper_2604_07239_b200.model import Predictor
from paper_2604_07239_b200.pipeline import StreamPartition
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 512
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0   # trained timesteps before the n profiled
cfg = ModelConfig(batch=batch, workers=1)
data = corpus.make_text(max(4_000_000, batch * (64 + skip + n)), 12)
part = StreamPartition.from_length(len(data), cfg.batch)
mat = np.ascontiguousarray(part.split(data)); L = part.stream_length
dmat = torch.from_numpy(mat).cuda()
m = Predictor(cfg)
lib = _native.lib(); coder = ctypes.c_void_p(); la = ctypes.c_int()
if skip:
    _native.check(lib.fade_bench_compress_steps(m.handle, dmat.data_ptr(), L, 16, skip, ctypes.byref(coder), ctypes.byref(la), None), "skip")
_native.check(lib.fade_bench_compress_steps(m.handle, dmat.data_ptr(), L, 16, n, ctypes.byref(coder), ctypes.byref(la), None), "steps")
torch.cuda.synchronize()
print("launches per timestep", la.value)
