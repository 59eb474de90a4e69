"""Predictor on the B200 vs the reference, from transplanted reference state.

Tolerances (north_star "stated tolerance"): the GEMMs run
on TF32 tensor cores, which TRUNCATE the operand mantissas to 10 bits.  The
activations that are only ever GEMM operands are stored already rounded to
nearest TF32 (x and h_mix through rounded copies), which leaves only the
weight operand truncated: tools/precision_study.py emulates that at KL
9.3e-7 / 3.9e-7 bits/symbol on the tiny / mid golden states (3.8e-6 / 1.5e-6
with both operands truncated), and the device measures 9.2e-7 / 4.1e-7.  So
one-step probabilities must match the reference within max-abs 1e-3 and mean
KL 1e-6 bits/symbol (SURVEY.md's proposed gate) -- about 1e-6 of a bit per
byte, far inside the 0.5% bits/byte gate; intermediates within 2e-3
relative to their scale; gradients within 2e-2 relative (TF32 through the
whole backward); one Adam step within 2.5*lr per element (Adam normalises,
so near-zero gradients may change sign) with a median far below lr.
"""

import numpy as np
import pytest

from conftest import model_golden

pytestmark = pytest.mark.gpu

PARTS = ("global", "local", "alpha", "mix", "mixer_inner", "coarse", "hidden", "logits")


def kl_bits(p, q):
    return float(np.mean(np.sum(p * (np.log2(p) - np.log2(q)), axis=1)))


def gpu_model(name):
    from paper_2604_07239_b200.model import Predictor
    cfg, st, z = model_golden(name)
    m = Predictor(cfg)
    m.load_state(st)
    return cfg, m, z


@pytest.mark.parametrize("name", ["tiny", "mid"])
def test_state_round_trip(name):
    cfg, m, z = gpu_model(name)
    s = m.save_state()
    for k, v in s["params"].items():
        np.testing.assert_array_equal(v, z["p_" + k], err_msg=k)
    np.testing.assert_array_equal(s["cache"], z["cache"])
    assert s["t"] == int(z["t"]) and s["step_count"] == int(z["step_count"])


@pytest.mark.parametrize("name", ["tiny", "mid"])
def test_forward_parts(name):
    cfg, m, z = gpu_model(name)
    parts = m.forward_debug(z["ctx"])
    for k in PARTS:
        ref = z["part_" + k]
        scale = max(1.0, float(np.abs(ref).max()))
        err = float(np.abs(parts[k] - ref).max()) / scale
        assert err < 2e-3, (k, err)
    # forward_debug touches no state
    np.testing.assert_array_equal(m.save_state()["cache"], z["cache"])


@pytest.mark.parametrize("name", ["tiny", "mid"])
def test_predict_probabilities(name):
    cfg, m, z = gpu_model(name)
    p = m.predict(z["ctx"])
    ref = z["next_probs"]
    assert np.abs(p - ref).max() < 1e-3
    assert kl_bits(ref, p) < 1e-6
    np.testing.assert_allclose(p.sum(axis=1), 1.0, atol=1e-12)
    assert (p > 0).all()
    assert 0.0 < m.alpha_stats[1] <= m.alpha_stats[0] <= m.alpha_stats[2] < 1.0


@pytest.mark.parametrize("name", ["tiny", "mid"])
def test_loss_and_gradients(name):
    from paper_2604_07239_b200.model import PARAM_ORDER
    cfg, m, z = gpu_model(name)
    loss, g = m.loss_grads(z["ctx"], z["tgt"])
    assert abs(loss - float(z["gloss"])) < 5e-3 * abs(float(z["gloss"]))
    for k in PARAM_ORDER:
        ref = z["g_" + k]
        scale = max(1e-12, float(np.abs(ref).max()))
        err = float(np.abs(g[k] - ref).max()) / scale
        # the residual weights' gradients are single sums over B*H products with
        # heavy cancellation, so their relative TF32 error is larger
        assert err < (1e-1 if ref.ndim == 0 else 2e-2), (k, err)
    # state untouched
    np.testing.assert_array_equal(m.save_state()["params"]["w_f"], z["p_w_f"])


@pytest.mark.parametrize("name", ["tiny", "mid"])
def test_one_train_step(name):
    from paper_2604_07239_b200.model import PARAM_ORDER
    cfg, m, z = gpu_model(name)
    m.predict(z["ctx"])
    m.train_step(z["tgt"])
    s = m.save_state()
    lr = cfg.lr
    for k in PARAM_ORDER:
        d = np.abs(s["params"][k] - z["next_p_" + k])
        assert d.max() <= 2.5 * lr, (k, d.max())
        assert np.median(d) <= 0.1 * lr, (k, np.median(d))
    assert s["t"] == int(z["t"]) + 1 and s["step_count"] == int(z["step_count"]) + 1
    np.testing.assert_allclose(s["cache"], z["next_cache"], atol=2e-3)


def test_trajectory_from_seeded_init():
    """40 online steps from the seeded init track the reference's probabilities."""
    from paper_2604_07239_b200.model import Predictor
    cfg, _, z = model_golden("tiny")
    m = Predictor(cfg)
    mat, t = z["mat"], cfg.ctx_len
    for j in range(z["probs"].shape[0]):
        i = t + j
        p = m.predict(mat[:, i - t:i])
        assert np.abs(p - z["probs"][j]).max() < 2e-2, j
        loss = m.train_step(mat[:, i])
        assert abs(loss - z["losses"][j]) < 2e-2, j


def test_train_without_predict_rejected():
    from paper_2604_07239_b200.model import Predictor
    cfg, _, _ = model_golden("tiny")
    m = Predictor(cfg)
    with pytest.raises(AssertionError):
        m.train_step(np.zeros(cfg.batch, np.uint8))
