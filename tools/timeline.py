"""In-graph kernel timeline of the compression timestep (CUPTI via
torch.profiler): per-kernel start offset, duration and stream for one
timestep, plus per-kernel mean durations over the profiled steps.

    python tools/timeline.py [steps] [batch] [skip] > timeline.txt

(skip: timesteps trained before the profiled ones; per-step cost grows a few
percent over the first ~10^4 steps of a stream)
"""
import ctypes
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from torch.profiler import ProfilerActivity, profile
    from paper_2604_07239_b200 import ModelConfig, _native, corpus
    from paper_2604_07239_b200.model import Predictor
    from paper_2604_07239_b200.pipeline import StreamPartition
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    batch = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    skip = int(sys.argv[3]) if len(sys.argv) > 3 else 32
    cfg = ModelConfig(batch=batch, workers=1)
    data = corpus.make_text(max(2_000_000, batch * (n + skip + 80)), 12)
    part = StreamPartition.from_length(len(data), cfg.batch)
    mat = np.ascontiguousarray(part.split(data))
    L = part.stream_length
    dmat = torch.from_numpy(mat).cuda()
    m = Predictor(cfg)
    lib = _native.lib()
    coder, la = ctypes.c_void_p(), ctypes.c_int()

    def steps(k):
        _native.check(lib.fade_bench_compress_steps(m.handle, dmat.data_ptr(), L, 16, k,
                                                    ctypes.byref(coder), ctypes.byref(la), None),
                      "steps")
    steps(skip)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        steps(n)
        torch.cuda.synchronize()
    path = os.path.join(tempfile.mkdtemp(), "trace.json")
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"]
          if e.get("cat") == "kernel" and e.get("ph") == "X"]
    ev.sort(key=lambda e: e["ts"])
    names = [e["name"] for e in ev]
    # one timestep = from a k_trunk_fwd to the next
    starts = [i for i, nm in enumerate(names) if nm.startswith(("void fade::k_trunk_fwd", "fade::k_trunk_fwd"))]
    if len(starts) < 3:
        print("no timesteps found", len(ev))
        return
    per_step = [(ev[starts[i + 1]]["ts"] - ev[starts[i]]["ts"]) for i in range(len(starts) - 1)]
    print(f"timesteps {len(per_step)}  mean {np.mean(per_step):.1f} us  min {min(per_step):.1f}")
    i0, i1 = starts[len(starts) // 2], starts[len(starts) // 2 + 1]
    t0 = ev[i0]["ts"]
    print(f"{'start':>8} {'dur':>7} {'end':>8} strm  kernel")
    for e in ev[i0:i1 + 1]:
        nm = e["name"].replace("void ", "").replace("fade::", "")[:60]
        print(f"{e['ts'] - t0:8.1f} {e['dur']:7.1f} {e['ts'] + e['dur'] - t0:8.1f} {e['args'].get('stream', '?'):>4}  {nm}")


if __name__ == "__main__":
    main()
