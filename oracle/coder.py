"""TEST INFRASTRUCTURE ONLY: ctypes front of ``oracle/coder_oracle.c``.

Same call convention as the reference kernel table
(``pkg/src/dszip/kernels.py:236-254``): numpy int64 arrays mutated in place,
rows ``[r0, r1)``, return -1 or the first failing row.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


def build() -> str:
    src = os.path.join(_HERE, "coder_oracle.c")
    if (not os.path.exists(_LIB_PATH)
            or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src)):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        i64, p = ctypes.c_int64, ctypes.c_void_p
        _lib.oracle_quantize_rows.argtypes = [p, p, i64, i64, i64]
        _lib.oracle_encode_step.argtypes = [p, i64, p, p, p, p, p, p, i64, p, i64, i64]
        _lib.oracle_flush.argtypes = [p, p, p, p, i64, p, i64, i64]
        _lib.oracle_prime.argtypes = [p, p, p, p, p, p, i64, i64]
        _lib.oracle_decode_step.argtypes = [p, i64, p, p, p, p, p, p, p, i64, i64, p]
        for f in ("oracle_quantize_rows", "oracle_encode_step", "oracle_flush",
                  "oracle_prime", "oracle_decode_step"):
            getattr(_lib, f).restype = i64
    return _lib


def _p(a: np.ndarray):
    assert a.flags.c_contiguous, "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(ctypes.c_void_p)


def quantize_rows(probs, freq, r0, r1) -> int:
    probs = np.ascontiguousarray(probs, dtype=np.float64)
    assert freq.dtype == np.int64
    return int(lib().oracle_quantize_rows(_p(probs), _p(freq), probs.shape[1], r0, r1))


def encode_step(cum, syms, low, rng, cache, ncache, buf, blen, r0, r1) -> int:
    cum = np.ascontiguousarray(cum, dtype=np.int64)
    syms = np.ascontiguousarray(syms, dtype=np.int64)
    return int(lib().oracle_encode_step(_p(cum), cum.shape[1], _p(syms), _p(low), _p(rng),
                                        _p(cache), _p(ncache), _p(buf), buf.shape[1],
                                        _p(blen), r0, r1))


def flush(low, cache, ncache, buf, blen, r0, r1) -> int:
    return int(lib().oracle_flush(_p(low), _p(cache), _p(ncache), _p(buf), buf.shape[1],
                                  _p(blen), r0, r1))


def prime(payload, off, dlen, pos, code, rng, r0, r1) -> int:
    payload = np.ascontiguousarray(payload, dtype=np.uint8)
    return int(lib().oracle_prime(_p(payload), _p(off), _p(dlen), _p(pos), _p(code),
                                  _p(rng), r0, r1))


def decode_step(cum, payload, off, dlen, pos, code, rng, out, r0, r1):
    cum = np.ascontiguousarray(cum, dtype=np.int64)
    payload = np.ascontiguousarray(payload, dtype=np.uint8)
    why = np.zeros(1, dtype=np.int64)
    k = int(lib().oracle_decode_step(_p(cum), cum.shape[1], _p(payload), _p(off), _p(dlen),
                                     _p(pos), _p(code), _p(rng), _p(out), r0, r1, _p(why)))
    return k, int(why[0])


TABLE = {
    "quantize_rows": quantize_rows,
    "encode_step": encode_step,
    "flush": flush,
    "prime": prime,
    "decode_step": decode_step,
}


# -- convenience wrappers used by the oracle pipeline -----------------------

def quantize(probs: np.ndarray) -> np.ndarray:
    freq = np.empty(probs.shape, dtype=np.int64)
    bad = quantize_rows(probs, freq, 0, probs.shape[0])
    if bad >= 0:
        raise ValueError(f"row {bad} does not sum to 1 within quantizer tolerance")
    return freq


def cum_from_freq(freq: np.ndarray) -> np.ndarray:
    cum = np.zeros((freq.shape[0], 257), dtype=np.int64)
    np.cumsum(freq, axis=1, out=cum[:, 1:])
    return cum


def uniform_cum(n: int) -> np.ndarray:
    return np.tile(np.arange(257, dtype=np.int64) * 256, (n, 1))


class Encoder:
    """Preallocated encoder state for ``n`` streams of at most ``steps`` symbols."""

    def __init__(self, n: int, steps: int):
        self.n = n
        self.low = np.zeros(n, np.int64)
        self.rng = np.full(n, 0xFFFFFFFF, np.int64)
        self.cache = np.zeros(n, np.int64)
        self.ncache = np.zeros(n, np.int64)
        self.buf = np.zeros((n, 2 * steps + 16), np.uint8)
        self.blen = np.zeros(n, np.int64)

    def encode(self, cum, syms):
        bad = encode_step(cum, syms, self.low, self.rng, self.cache, self.ncache,
                          self.buf, self.blen, 0, self.n)
        if bad >= 0:
            raise ValueError(f"zero-frequency symbol in stream {bad}")

    def finish(self) -> list:
        flush(self.low, self.cache, self.ncache, self.buf, self.blen, 0, self.n)
        return [self.buf[k, :self.blen[k]].tobytes() for k in range(self.n)]


class Decoder:
    def __init__(self, payload, offsets, lengths):
        self.payload = np.ascontiguousarray(payload, dtype=np.uint8)
        self.off = np.ascontiguousarray(offsets, dtype=np.int64)
        self.dlen = np.ascontiguousarray(lengths, dtype=np.int64)
        n = len(self.off)
        self.n = n
        self.pos = np.zeros(n, np.int64)
        self.code = np.zeros(n, np.int64)
        self.rng = np.zeros(n, np.int64)
        bad = prime(self.payload, self.off, self.dlen, self.pos, self.code, self.rng, 0, n)
        if bad >= 0:
            raise ValueError(f"stream {bad} shorter than the coder tail")

    def decode(self, cum) -> np.ndarray:
        out = np.zeros(self.n, np.int64)
        k, why = decode_step(cum, self.payload, self.off, self.dlen, self.pos, self.code,
                             self.rng, out, 0, self.n)
        if k >= 0:
            raise ValueError(f"stream {k}: {'truncated' if why == 2 else 'invalid code'}")
        return out
