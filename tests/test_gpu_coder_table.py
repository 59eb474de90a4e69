"""Kernel-table entries on the GPU vs the reference's golden tables and
bitstreams (bit-exact), through the C ABI on device arrays."""

import numpy as np
import pytest

from conftest import load_golden

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_quantizer_bit_exact():
    from paper_2604_07239_b200 import _native
    lib = _native.lib()
    z = load_golden("quant.npz")
    p = dev(z["probs"])
    f = torch.zeros(p.shape, dtype=torch.int64, device="cuda")
    assert lib.fade_quantize_rows(p.data_ptr(), f.data_ptr(), 0, p.shape[0], None) == -1
    np.testing.assert_array_equal(f.cpu().numpy(), z["freq"])


def test_quantizer_reports_first_bad_row():
    from paper_2604_07239_b200 import _native
    lib = _native.lib()
    z = load_golden("quant.npz")
    p = dev(z["bad_probs"])
    f = torch.zeros(p.shape, dtype=torch.int64, device="cuda")
    assert lib.fade_quantize_rows(p.data_ptr(), f.data_ptr(), 0, 3, None) == int(z["bad_row"])


def encode_all(cums, syms, cap):
    from paper_2604_07239_b200 import _native
    lib = _native.lib()
    steps, rows = syms.shape
    low = torch.zeros(rows, dtype=torch.int64, device="cuda")
    rng = torch.full((rows,), 0xFFFFFFFF, dtype=torch.int64, device="cuda")
    cache = torch.zeros_like(low)
    ncache = torch.zeros_like(low)
    blen = torch.zeros_like(low)
    buf = torch.zeros((rows, cap), dtype=torch.uint8, device="cuda")
    cd = dev(cums.astype(np.int64))
    sd = dev(syms.astype(np.int64))
    for i in range(steps):
        k = lib.fade_encode_step(cd[i].data_ptr(), 257, sd[i].data_ptr(), low.data_ptr(),
                                 rng.data_ptr(), cache.data_ptr(), ncache.data_ptr(),
                                 buf.data_ptr(), cap, blen.data_ptr(), 0, rows, None)
        assert k == -1
    assert lib.fade_flush(low.data_ptr(), cache.data_ptr(), ncache.data_ptr(), buf.data_ptr(), cap,
                          blen.data_ptr(), 0, rows, None) == -1
    b = buf.cpu().numpy()
    n = blen.cpu().numpy()
    return [b[k, :n[k]].tobytes() for k in range(rows)]


def test_encoder_bitstreams_bit_exact():
    z = load_golden("coder.npz")
    streams = encode_all(z["cums"], z["syms"], 2 * z["syms"].shape[0] + 16)
    assert [len(s) for s in streams] == list(z["lengths"])
    assert b"".join(streams) == z["payload"].tobytes()


def test_encoder_first_byte_quirk():
    z = load_golden("coder.npz")
    streams = encode_all(z["quirk_cums"], z["quirk_syms"], 32)
    assert b"".join(streams) == z["quirk_payload"].tobytes()


def test_decoder_bit_exact_and_truncation():
    from paper_2604_07239_b200 import _native
    lib = _native.lib()
    z = load_golden("coder.npz")
    cums, syms = z["cums"].astype(np.int64), z["syms"].astype(np.int64)
    rows = syms.shape[1]
    lengths = z["lengths"].astype(np.int64)
    offs = np.concatenate([[0], np.cumsum(lengths)[:-1]]).astype(np.int64)
    for trunc in (False, True):
        dlen = lengths.copy()
        if trunc:
            dlen[5] = 7
        pay, off, dl = dev(z["payload"]), dev(offs), dev(dlen)
        pos = torch.zeros(rows, dtype=torch.int64, device="cuda")
        code = torch.zeros_like(pos)
        rng = torch.zeros_like(pos)
        assert lib.fade_prime(pay.data_ptr(), off.data_ptr(), dl.data_ptr(), pos.data_ptr(),
                              code.data_ptr(), rng.data_ptr(), 0, rows, None) == -1
        out = torch.zeros_like(pos)
        cd = dev(cums)
        failed = None
        for i in range(len(syms)):
            why = _native.i64(0)
            k = lib.fade_decode_step(cd[i].data_ptr(), 257, pay.data_ptr(), off.data_ptr(),
                                     dl.data_ptr(), pos.data_ptr(), code.data_ptr(),
                                     rng.data_ptr(), out.data_ptr(), 0, rows,
                                     _native.ctypes.byref(why), None)
            if k >= 0:
                failed = (k, why.value)
                break
            np.testing.assert_array_equal(out.cpu().numpy(), syms[i])
        if trunc:
            assert failed is not None and failed[0] == 5 and failed[1] == 2
        else:
            assert failed is None


def test_prime_rejects_short_stream():
    from paper_2604_07239_b200 import _native
    lib = _native.lib()
    pay = dev(np.arange(32, dtype=np.uint8))
    off = dev(np.array([0, 8, 16], np.int64))
    dl = dev(np.array([8, 3, 8], np.int64))
    pos = torch.zeros(3, dtype=torch.int64, device="cuda")
    code = torch.zeros_like(pos)
    rng = torch.zeros_like(pos)
    assert lib.fade_prime(pay.data_ptr(), off.data_ptr(), dl.data_ptr(), pos.data_ptr(),
                          code.data_ptr(), rng.data_ptr(), 0, 3, None) == 1
    assert code[0].item() == 0x00010203 and code[2].item() == 0 and pos[2].item() == 0
