"""Loader for the sm_100a extension ``_lib/libfade_b200.so`` (ctypes, C ABI).

There is deliberately no fallback: if the library or a CUDA device is missing,
``lib()`` raises and every product entry point fails loudly.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libfade_b200.so")
# (FADE_LIB_PATH points at an alternative build of the same library: A/B timing)
LIB_PATH = os.environ.get("FADE_LIB_PATH", LIB_PATH)

_lib = None

i32, i64, f64, vp = ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
P = ctypes.POINTER


class FadeError(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("why", ctypes.c_int32),
                ("stream", ctypes.c_int64), ("step", ctypes.c_int64)]


class FadeConfig(ctypes.Structure):
    _fields_ = [("ctx_len", ctypes.c_int32), ("embed_dim", ctypes.c_int32),
                ("cache_dim", ctypes.c_int32), ("mix_dim", ctypes.c_int32),
                ("expand_dim", ctypes.c_int32), ("batch", ctypes.c_int32),
                ("alphabet", ctypes.c_int32), ("conv_kernel", ctypes.c_int32),
                ("lr", ctypes.c_double), ("beta1", ctypes.c_double),
                ("beta2", ctypes.c_double), ("adam_eps", ctypes.c_double),
                ("variant", ctypes.c_int32)]


# name -> (restype, argtypes); must match include/fade_b200.h
SIGNATURES = {
    "fade_last_error": (ctypes.c_char_p, []),
    "fade_abi_version": (i32, []),
    "fade_device_count": (i32, []),
    "fade_device_arch": (i32, [i32, P(i32), P(i32), ctypes.c_char_p, i32]),
    "fade_quantize_rows": (i64, [vp, vp, i64, i64, vp]),
    "fade_encode_step": (i64, [vp, i64, vp, vp, vp, vp, vp, vp, i64, vp, i64, i64, vp]),
    "fade_flush": (i64, [vp, vp, vp, vp, i64, vp, i64, i64, vp]),
    "fade_prime": (i64, [vp, vp, vp, vp, vp, vp, i64, i64, vp]),
    "fade_decode_step": (i64, [vp, i64, vp, vp, vp, vp, vp, vp, vp, i64, i64, P(i64), vp]),
    "fade_model_create": (i32, [P(FadeConfig), i32, P(vp)]),
    "fade_model_destroy": (i32, [vp]),
    "fade_model_set_tensor": (i32, [vp, i32, i32, vp, i64]),
    "fade_model_get_tensor": (i32, [vp, i32, i32, vp, i64]),
    "fade_model_set_cache": (i32, [vp, vp]),
    "fade_model_get_cache": (i32, [vp, vp]),
    "fade_model_set_counters": (i32, [vp, i64, i64]),
    "fade_model_get_counters": (i32, [vp, P(i64), P(i64)]),
    "fade_model_predict": (i32, [vp, vp, vp, vp, P(FadeError)]),
    "fade_model_train_step": (i32, [vp, vp, P(f64), P(FadeError)]),
    "fade_model_forward_debug": (i32, [vp, vp, ctypes.c_char_p, vp]),
    "fade_model_loss_grads": (i32, [vp, vp, vp, P(f64)]),
    "fade_compress": (i32, [vp, i32, i32, vp, i64, i64, i32, i32, vp, vp, vp, vp, P(vp),
                            P(FadeError)]),
    "fade_coder_fetch": (i32, [vp, vp, i64]),
    "fade_coder_destroy": (i32, [vp]),
    "fade_decompress": (i32, [vp, i32, i32, vp, i64, vp, i64, i64, vp, vp, vp, vp, P(FadeError)]),
    "fade_bench_compress_steps": (i32, [vp, vp, i64, i64, i64, P(vp), P(i32), vp]),
    "fade_model_stream": (i32, [vp, P(vp)]),
    "fade_bench_probe": (i32, [vp, i32, i32, P(f64), P(f64), P(f64)]),
    "fade_debug_gemm": (i32, [vp, i64, i32, vp, i64, i32, vp, i64, i32, i32, i32, i32, i32, i32,
                              vp]),
}


def lib():
    """Load the extension (raises OSError if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OSError(f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build())")
        so = ctypes.CDLL(LIB_PATH)
        missing = [n for n in SIGNATURES if not hasattr(so, n)]
        if missing:
            raise OSError(f"{LIB_PATH} lacks exports {missing}: rebuild it")
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(so, name)
            fn.restype = res
            fn.argtypes = args
        _lib = so
    return _lib


def last_error() -> str:
    msg = lib().fade_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str) -> None:
    if status != 0:
        raise RuntimeError(f"{what} failed (status {status}): {last_error()}")


_BUILD_ID = None


def build_id() -> str:
    """First 16 hex digits of the loaded library's sha256: identifies the exact
    kernels (and so the float trajectory) that wrote a container."""
    global _BUILD_ID
    if _BUILD_ID is None:
        import hashlib
        with open(LIB_PATH, "rb") as fh:
            _BUILD_ID = hashlib.sha256(fh.read()).hexdigest()[:16]
    return _BUILD_ID


def device_arch(device: int) -> str:
    """e.g. 'sm_100 NVIDIA B200' for the given CUDA device."""
    ma, mi = ctypes.c_int(), ctypes.c_int()
    name = ctypes.create_string_buffer(128)
    check(lib().fade_device_arch(int(device), ctypes.byref(ma), ctypes.byref(mi), name, 128),
          "fade_device_arch")
    return f"sm_{ma.value}{mi.value} {name.value.decode()}"


def require_device() -> None:
    """Fail loudly when no CUDA device is visible (no CPU fallback exists)."""
    n = lib().fade_device_count()
    if n < 1:
        raise RuntimeError("paper_2604_07239_b200 needs a CUDA device (B200, sm_100a); none visible")
