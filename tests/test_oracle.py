"""Pin the CPU oracle against golden vectors produced by the reference itself.

The oracle is the checker for every GPU parity test, so it must first agree
with the reference: bit-exactly on the integer path, and to float32 rounding
noise on the model (the golden states come from the reference's numpy run).
"""

import hashlib
import json

import numpy as np
import pytest

from conftest import golden_json, load_golden, model_golden
from oracle import coder as oc
from oracle.model import PARAM_ORDER, OracleModel, init_params, softmax64, softmax_xent


class TestCoderOracle:
    def test_quantizer_matches_reference(self):
        z = load_golden("quant.npz")
        freq = np.empty(z["probs"].shape, np.int64)
        assert oc.quantize_rows(z["probs"], freq, 0, len(freq)) == -1
        np.testing.assert_array_equal(freq, z["freq"])
        assert (freq.sum(axis=1) == 65536).all() and freq.min() >= 1

    def test_quantizer_error_row(self):
        z = load_golden("quant.npz")
        fb = np.empty(z["bad_probs"].shape, np.int64)
        assert oc.quantize_rows(z["bad_probs"], fb, 0, 3) == int(z["bad_row"])

    def test_encoder_bitstreams_bit_exact(self):
        z = load_golden("coder.npz")
        cums, syms = z["cums"].astype(np.int64), z["syms"].astype(np.int64)
        steps, rows = syms.shape
        enc = oc.Encoder(rows, steps)
        for i in range(steps):
            enc.encode(cums[i], syms[i])
        streams = enc.finish()
        assert [len(s) for s in streams] == list(z["lengths"])
        assert b"".join(streams) == z["payload"].tobytes()

    def test_decoder_round_trip(self):
        z = load_golden("coder.npz")
        cums, syms = z["cums"].astype(np.int64), z["syms"].astype(np.int64)
        lengths = z["lengths"]
        offs = np.concatenate([[0], np.cumsum(lengths)[:-1]]).astype(np.int64)
        dec = oc.Decoder(z["payload"], offs, lengths)
        for i in range(len(syms)):
            np.testing.assert_array_equal(dec.decode(cums[i]), syms[i])

    def test_first_byte_quirk_reproduced(self):
        z = load_golden("coder.npz")
        rows = z["quirk_syms"].shape[1]
        enc = oc.Encoder(rows, 4)
        for i in range(2):
            enc.encode(z["quirk_cums"][i], z["quirk_syms"][i])
        out = enc.finish()
        assert b"".join(out) == z["quirk_payload"].tobytes()
        assert out[0][0] == 0x00     # the stale cache byte where 0xFF belongs

    def test_truncation_reported(self):
        z = load_golden("coder.npz")
        cums = z["cums"].astype(np.int64)
        lengths = z["lengths"].copy()
        offs = np.concatenate([[0], np.cumsum(lengths)[:-1]]).astype(np.int64)
        short = lengths.copy()
        short[3] = 6
        dec = oc.Decoder(z["payload"], offs, short)
        with pytest.raises(ValueError, match="stream 3"):
            for i in range(len(cums)):
                dec.decode(cums[i])


class TestModelOracle:
    @pytest.mark.parametrize("name", ["tiny", "mid"])
    def test_forward_parts(self, name):
        cfg, st, z = model_golden(name)
        m = OracleModel(cfg)
        m.load_state(st)
        logits, s = m.forward(z["ctx"])
        for key, ours in (("global", s["h_g"]), ("local", s["h_l"]), ("alpha", s["alpha"]),
                          ("mix", s["h_mix"]), ("mixer_inner", s["inner"]),
                          ("coarse", s["h_c"]), ("hidden", s["h"]), ("logits", logits)):
            ref = z["part_" + key]
            np.testing.assert_allclose(ours, ref, rtol=2e-5, atol=2e-6, err_msg=key)
        np.testing.assert_allclose(softmax64(logits), z["next_probs"], atol=1e-7)

    @pytest.mark.parametrize("name", ["tiny", "mid"])
    def test_gradients(self, name):
        cfg, st, z = model_golden(name)
        m = OracleModel(cfg)
        m.load_state(st)
        loss, g = m.loss_grads(z["ctx"], z["tgt"])
        assert abs(loss - float(z["gloss"])) < 1e-6
        for k in PARAM_ORDER:
            ref = z["g_" + k]
            scale = max(1e-12, float(np.abs(ref).max()))
            err = float(np.abs(g[k] - ref).max()) / scale
            assert err < 2e-4, (k, err)

    @pytest.mark.parametrize("name", ["tiny", "mid"])
    def test_train_step_updates(self, name):
        cfg, st, z = model_golden(name)
        m = OracleModel(cfg)
        m.load_state(st)
        m.predict(z["ctx"])
        m.train_step(z["tgt"])
        for k in PARAM_ORDER:
            np.testing.assert_allclose(m.p[k], z["next_p_" + k], rtol=1e-5, atol=2e-6,
                                       err_msg=k)
        np.testing.assert_allclose(m.cache, z["next_cache"], atol=1e-6)

    def test_trajectory_from_init(self):
        """From the seeded init, the oracle tracks the reference's probabilities."""
        cfg, _, z = model_golden("tiny")
        m = OracleModel(cfg)
        mat = z["mat"]
        t = cfg.ctx_len
        for j in range(z["probs"].shape[0]):
            i = t + j
            pr = m.predict(mat[:, i - t:i])
            assert np.abs(pr - z["probs"][j]).max() < 1e-4, j
            loss = m.train_step(mat[:, i])
            assert abs(loss - z["losses"][j]) < 1e-4, j

    def test_init_matches_reference_default_digest(self):
        from paper_2604_07239_b200.config import ModelConfig
        z = load_golden("model_default_digest.npz")
        dig = json.loads(bytes(z["digest_json"]).decode())
        p = init_params(ModelConfig(seed=5))
        for k in PARAM_ORDER:
            assert hashlib.sha256(p[k].tobytes()).hexdigest() == dig[k], k


def _tf32(a, mode):
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    if mode == "rne":
        u = u + 0xFFF + ((u >> 13) & 1)
    return (u & 0xFFFFE000).astype(np.uint32).view(np.float32)


class _TF32(np.ndarray):
    mode = "trunc"

    def __matmul__(self, other):
        return np.matmul(_tf32(np.asarray(self), _TF32.mode), _tf32(np.asarray(other), _TF32.mode))

    def __rmatmul__(self, other):
        return np.matmul(_tf32(np.asarray(other), _TF32.mode), _tf32(np.asarray(self), _TF32.mode))


@pytest.mark.parametrize("name", ["tiny", "mid"])
def test_tf32_truncation_budget(name):
    """The GPU gate in test_gpu_model.py is derived here: emulate TF32 operand
    truncation (what tcgen05.kind::tf32 does) on the golden state and measure
    the probability error against the reference."""
    cfg, st, z = model_golden(name)
    out = {}
    for mode in ("trunc", "rne"):
        m = OracleModel(cfg)
        m.load_state(st)
        _TF32.mode = mode
        for k in list(m.p):
            m.p[k] = m.p[k].view(_TF32)
        m.cache = m.cache.view(_TF32)
        lg, _ = m.forward(z["ctx"])
        p = softmax64(np.asarray(lg))
        ref = z["next_probs"]
        kl = float(np.mean(np.sum(ref * (np.log2(ref) - np.log2(p)), axis=1)))
        out[mode] = (float(np.abs(p - ref).max()), kl)
    assert out["trunc"][0] < 1e-3 and out["trunc"][1] < 1e-5
    assert out["rne"][1] < out["trunc"][1]


def test_softmax_xent_grad_is_p_minus_onehot():
    rng = np.random.default_rng(0)
    lg = rng.normal(size=(8, 256)).astype(np.float32)
    tg = rng.integers(0, 256, 8)
    loss, d = softmax_xent(lg, tg)
    p = softmax64(lg)
    p[np.arange(8), tg] -= 1
    np.testing.assert_allclose(d, (p / 8).astype(np.float32))
    assert loss > 0


def test_bpb_fixture_has_reference_sizes():
    sizes = golden_json("bpb.json")
    assert sizes["default_text1m"]["bytes"] == 233320
    assert all(v["bytes"] > 0 for v in sizes.values())


def test_torch_oracle_tracks_reference_trajectory():
    """oracle/torch_model.py (the large-size bits/byte oracle, fp32 autograd +
    the reference's Adam) reproduces the reference's 40-step trajectory from
    the seeded init, on CPU here (the GPU runs it with TF32 disabled)."""
    from oracle.torch_model import TorchOracle
    cfg, _, z = model_golden("tiny")
    m = TorchOracle(cfg, device="cpu")
    mat, t = z["mat"], cfg.ctx_len
    for j in range(z["probs"].shape[0]):
        i = t + j
        p = m.predict(mat[:, i - t:i]).numpy()
        assert np.abs(p - z["probs"][j]).max() < 1e-4, j
        loss = m.train_step(mat[:, i])
        assert abs(loss - z["losses"][j]) < 1e-4, j
