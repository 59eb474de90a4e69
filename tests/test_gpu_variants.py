"""Ablation variants (model.py:39, 121-175) on the B200 vs the reference's own
trajectories (tests/golden/variants.npz, made by tests/golden/make_golden.py):
from the same seeded init, 12 predict/train steps -- probabilities, losses
and router statistics per step -- then the loss gradients of every parameter.
Tolerances are the TF32 ones of tests/test_gpu_model.py."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

VARIANTS = ("full", "dual", "global_only", "local_only", "mixer_nogate", "mixer")


def _cfg():
    from paper_2604_07239_b200 import ModelConfig
    return ModelConfig(ctx_len=4, embed_dim=8, cache_dim=32, mix_dim=8, expand_dim=32,
                       batch=16, workers=1, seed=9)


@pytest.mark.parametrize("variant", VARIANTS)
def test_variant_trajectory_and_grads(variant):
    from paper_2604_07239_b200.model import PARAM_ORDER, Predictor
    z = load_golden("variants.npz")
    mat = z["mat"]
    cfg = _cfg()
    m = Predictor(cfg, variant)
    t = cfg.ctx_len
    ref_p, ref_l, ref_a = z[variant + "__probs"], z[variant + "__losses"], z[variant + "__alphas"]
    for k in range(len(ref_l)):
        i = t + k
        p = m.predict(mat[:, i - t:i])
        assert np.abs(p[:8] - ref_p[k]).max() < 1e-3, (variant, k)
        if np.isnan(ref_a[k, 0]):
            assert m.alpha_stats is None
        else:
            assert np.allclose(m.alpha_stats, ref_a[k], atol=1e-3), (variant, k)
        loss = m.train_step(mat[:, i])
        assert abs(loss - ref_l[k]) < 2e-3 * abs(ref_l[k]), (variant, k, loss, ref_l[k])
    i = t + len(ref_l)
    loss, grads = m.loss_grads(mat[:, i - t:i], mat[:, i])
    assert abs(loss - float(z[variant + "__gloss"])) < 2e-3 * abs(float(z[variant + "__gloss"]))
    for name in PARAM_ORDER:
        ref = z[variant + "__g_" + name]
        got = grads[name].reshape(ref.shape)
        scale = max(np.abs(ref).max(), 1e-12)
        if np.abs(ref).max() == 0.0:
            assert np.abs(got).max() == 0.0, (variant, name)       # unused by this variant
        else:
            tol = 0.1 if ref.size == 1 else 2e-2
            assert np.abs(got - ref).max() / scale < tol, (variant, name)


@pytest.mark.parametrize("variant", ("dual", "global_only", "local_only", "mixer_nogate", "mixer"))
def test_variant_compress_and_metrics(variant):
    """run_ablation's path (bench.py:142-180): the pipelined executor compresses
    with an ablation model; the metrics tape carries router statistics only
    for the routed variants (model.py:146-151)."""
    from paper_2604_07239_b200 import corpus
    from paper_2604_07239_b200.pipeline import run_pipelined_compress
    data = corpus.make_text(2000, 5)
    res = run_pipelined_compress(data, _cfg(), variant=variant, collect_metrics=True)
    assert len(res.losses) > 0 and all(np.isfinite(res.losses))
    has_alpha = variant not in ("global_only", "local_only")
    assert ("alpha_mean" in res.metrics[0]) == has_alpha


def test_run_ablation_and_sweep(tmp_path):
    """bench.py:99-180 harnesses over the device executors."""
    from paper_2604_07239_b200 import corpus, harness
    from paper_2604_07239_b200.model import Predictor
    data = corpus.make_text(3000, 6)
    rep = harness.run_ablation(data, _cfg())
    assert set(rep) == set(VARIANTS)
    full_params = Predictor(_cfg()).param_count()
    for v, r in rep.items():
        assert r["steps"] > 0 and 0.0 < r["bits_per_byte"] < 10.0 and r["ratio"] > 0.0
        assert 0 < r["active_params"] <= full_params
    assert rep["full"]["active_params"] == full_params
    paths = []
    for k, kind in enumerate(("text", "dna")):
        p = tmp_path / f"f{k}.bin"
        p.write_bytes(getattr(corpus, "make_" + kind)(2500, k + 1))
        paths.append(p)
    sw = harness.run_sweep(paths, _cfg())
    assert len(sw["files"]) == 2
    assert all(0.0 <= r["score"] <= 1.0 for r in sw["files"])


ROW_PROBE = """
import json, sys
import numpy as np
sys.path.insert(0, {root!r})
from paper_2604_07239_b200 import ModelConfig, corpus
from paper_2604_07239_b200.model import Predictor
cfg = ModelConfig(batch=64, workers=1, seed=4, **{dims!r})
T = cfg.ctx_len
mat = np.frombuffer(corpus.make_text(64 * (T + 6), 3), np.uint8).reshape(64, T + 6)
out = {{}}
for v in {variants!r}:
    m = Predictor(cfg, v)
    rows = []
    for i in range(T, T + 6):
        p = m.predict(mat[:, i - T:i])
        rows.append([p[:4].tolist(), m.train_step(mat[:, i])])
    out[v] = rows
print(json.dumps(out))
"""


@pytest.mark.parametrize("dims", [
    dict(ctx_len=8, embed_dim=16, cache_dim=256, mix_dim=32, expand_dim=256),
    # H = 512 at D = 32, T = 16, K = 3: also the warp-per-row trunk forward
    dict(ctx_len=16, embed_dim=32, cache_dim=512, mix_dim=32, expand_dim=512)])
def test_warp_and_cta_row_kernels_agree_on_every_variant(dims):
    """The warp-per-row kernels (row_warp.cu, used from B = 2048) and the
    CTA-per-row kernels compute the same thing for every variant's flags:
    the experiments build runs both (FADE_ROW_WARP = 255 / 0) and the
    trajectories agree to fp32 reduction-order noise."""
    import json
    import os
    import subprocess
    import sys
    from conftest import ROOT
    lib = os.path.join(ROOT, "build", "exp", "libfade_b200.so")
    if not os.path.exists(lib):
        pytest.skip("experiments build (make experiments) not present")
    code = ROW_PROBE.format(root=ROOT, variants=VARIANTS, dims=dims)
    res = {}
    for mask in ("0", "255"):
        env = dict(os.environ, FADE_LIB_PATH=lib, FADE_ROW_WARP=mask)
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                             timeout=600)
        assert out.returncode == 0, out.stderr[-3000:]
        res[mask] = json.loads(out.stdout.strip().splitlines()[-1])
    for v in VARIANTS:
        for (p0, l0), (p1, l1) in zip(res["0"][v], res["255"][v]):
            assert np.abs(np.array(p0) - np.array(p1)).max() < 1e-4, v
            assert abs(l0 - l1) < 1e-4, v


WS_PROBE = """
import hashlib, sys
sys.path.insert(0, {root!r})
from paper_2604_07239_b200 import ModelConfig, container, corpus
data = corpus.make_text(64 * 200, 4)
blob, _ = container.compress_bytes(data, ModelConfig(seed=5, batch=64))
print(hashlib.sha256(blob).hexdigest())
"""


def test_persistent_adam_gemm_is_bit_identical():
    """The persistent warp-specialised GEMM's Adam epilogue (gemm_ws.cuh; the
    W12 update through it with FADE_WS, experiments build) runs the same MMA
    k order and the same Adam rounding sequence as the one-tile-per-CTA
    kernel: the containers are byte-identical."""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    lib = os.path.join(ROOT, "build", "exp", "libfade_b200.so")
    if not os.path.exists(lib):
        pytest.skip("experiments build (make experiments) not present")
    code = WS_PROBE.format(root=ROOT)
    out = {}
    for ws in ("8", "16392"):   # expand GEMM only / expand GEMM + W12 update
        env = dict(os.environ, FADE_LIB_PATH=lib, FADE_WS=ws)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        out[ws] = r.stdout.strip().splitlines()[-1]
    assert out["8"] == out["16392"]
