"""Kernel table: the reference's five integer kernels, backed by the B200.

Mirrors ``pkg/src/dszip/kernels.py:236-273``: ``BACKENDS[name]`` maps to a
dict of ``quantize_rows / encode_step / flush / prime / decode_step`` with the
reference signatures (numpy arrays mutated in place, rows ``[r0, r1)``,
return -1 or the first failing row).  The only backend here is ``"cuda"``:
arrays are staged to the device, the sm_100a kernels run, and results are
copied back.  ``DSZIP_BACKEND`` may name ``cuda``; anything else is rejected
exactly as the reference rejects an unknown backend.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _native

TOP = 1 << 24
MASK32 = (1 << 32) - 1
PRECISION = 16
TOTAL = 1 << PRECISION
HAS_NUMBA = False


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the cuda kernel backend needs a CUDA device (B200)")
    return torch


def _dev(a: np.ndarray):
    torch = _torch()
    a = np.ascontiguousarray(a)
    if not a.flags.writeable:          # torch refuses read-only numpy buffers
        a = a.copy()
    return torch.from_numpy(a).cuda()


def _back(t, out: np.ndarray) -> None:
    out[...] = t.cpu().numpy().reshape(out.shape)


def quantize_rows(probs, freq, r0, r1):
    p = _dev(np.asarray(probs, dtype=np.float64))
    f = _dev(freq)
    bad = _native.lib().fade_quantize_rows(p.data_ptr(), f.data_ptr(), r0, r1, None)
    if bad == -2:
        raise RuntimeError(_native.last_error())
    _back(f, freq)
    return int(bad)


def encode_step(cum, syms, low, rng, cache, ncache, buf, blen, r0, r1):
    c = _dev(np.asarray(cum, dtype=np.int64))
    s = _dev(np.asarray(syms, dtype=np.int64))
    st = [_dev(x) for x in (low, rng, cache, ncache, buf, blen)]
    bad = _native.lib().fade_encode_step(c.data_ptr(), c.shape[1], s.data_ptr(),
                                         st[0].data_ptr(), st[1].data_ptr(), st[2].data_ptr(),
                                         st[3].data_ptr(), st[4].data_ptr(), buf.shape[1],
                                         st[5].data_ptr(), r0, r1, None)
    if bad == -2:
        raise RuntimeError(_native.last_error())
    for t, x in zip(st, (low, rng, cache, ncache, buf, blen)):
        _back(t, x)
    return int(bad)


def flush(low, cache, ncache, buf, blen, r0, r1):
    st = [_dev(x) for x in (low, cache, ncache, buf, blen)]
    bad = _native.lib().fade_flush(st[0].data_ptr(), st[1].data_ptr(), st[2].data_ptr(),
                                   st[3].data_ptr(), buf.shape[1], st[4].data_ptr(), r0, r1, None)
    if bad == -2:
        raise RuntimeError(_native.last_error())
    for t, x in zip(st, (low, cache, ncache, buf, blen)):
        _back(t, x)
    return int(bad)


def prime(payload, off, dlen, pos, code, rng, r0, r1):
    pay = _dev(np.asarray(payload, dtype=np.uint8))
    o, d = _dev(np.asarray(off, np.int64)), _dev(np.asarray(dlen, np.int64))
    st = [_dev(x) for x in (pos, code, rng)]
    bad = _native.lib().fade_prime(pay.data_ptr(), o.data_ptr(), d.data_ptr(), st[0].data_ptr(),
                                   st[1].data_ptr(), st[2].data_ptr(), r0, r1, None)
    if bad == -2:
        raise RuntimeError(_native.last_error())
    for t, x in zip(st, (pos, code, rng)):
        _back(t, x)
    return int(bad)


def decode_step(cum, payload, off, dlen, pos, code, rng, out, r0, r1):
    c = _dev(np.asarray(cum, dtype=np.int64))
    pay = _dev(np.asarray(payload, dtype=np.uint8))
    o, d = _dev(np.asarray(off, np.int64)), _dev(np.asarray(dlen, np.int64))
    st = [_dev(x) for x in (pos, code, rng, out)]
    why = ctypes.c_int64(0)
    k = _native.lib().fade_decode_step(c.data_ptr(), c.shape[1], pay.data_ptr(), o.data_ptr(),
                                       d.data_ptr(), st[0].data_ptr(), st[1].data_ptr(),
                                       st[2].data_ptr(), st[3].data_ptr(), r0, r1,
                                       ctypes.byref(why), None)
    if k == -2:
        raise RuntimeError(_native.last_error())
    for t, x in zip(st, (pos, code, rng, out)):
        _back(t, x)
    return int(k), int(why.value)


BACKENDS: dict[str, dict] = {
    "cuda": {
        "quantize_rows": quantize_rows,
        "encode_step": encode_step,
        "flush": flush,
        "prime": prime,
        "decode_step": decode_step,
    }
}


def _pick_backend() -> str:
    want = os.environ.get("DSZIP_BACKEND", "").strip().lower()
    if want and want not in BACKENDS:
        raise RuntimeError(f"DSZIP_BACKEND={want!r} unavailable (have: {', '.join(BACKENDS)})")
    return "cuda"


BACKEND = _pick_backend()
