"""Executors: stream partitioning, serial / pipelined compression and
decompression, all running the whole timestep loop on the B200.

Keeps the reference executor API (``pkg/src/dszip/pipeline.py:35-411``).  The
difference is where the loop lives: the reference runs predict -> quantise ->
encode -> train as Python calls on two host threads (model / coder) around a
two-slot ping-pong buffer; here one ``fade_compress`` / ``fade_decompress`` call
replays a captured CUDA graph per timestep.  The pipelined executor puts the
encoder on its own CUDA stream, draining the step's cumulative-table slot while
the model stream runs the backward pass -- the same two-slot protocol
(empty -> filling -> full -> draining -> empty) enforced by CUDA events instead
of a ``threading.Condition``.  Serial and pipelined produce identical bytes
because the table for step i is always built before the step-i update.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .config import ModelConfig
from .errors import CorruptionError, ModelDivergenceError
from .model import LN2, Predictor, default_device

__all__ = [
    "StreamPartition",
    "PingPongBuffer",
    "CompressResult",
    "run_serial_compress",
    "run_pipelined_compress",
    "run_parallel_decompress",
    "throughput_report",
]


@dataclass(frozen=True)
class StreamPartition:
    """Flat bytes <-> (n_streams, stream_length) grid (pipeline.py:35-64).

    Stream k covers bytes [k*L, (k+1)*L); the last stream is zero padded.
    """

    original_length: int
    n_streams: int
    stream_length: int

    @classmethod
    def from_length(cls, length: int, n_streams: int) -> "StreamPartition":
        return cls(length, n_streams, -(-length // n_streams) if length else 0)

    @property
    def pad(self) -> int:
        return self.n_streams * self.stream_length - self.original_length

    def split(self, data: bytes) -> np.ndarray:
        if len(data) != self.original_length:
            raise ValueError("data length does not match partition")
        grid = np.zeros(self.n_streams * self.stream_length, dtype=np.uint8)
        grid[:self.original_length] = np.frombuffer(data, dtype=np.uint8)
        return grid.reshape(self.n_streams, self.stream_length)

    def join(self, mat: np.ndarray) -> bytes:
        return mat.reshape(-1)[:self.original_length].tobytes()


_LEGAL = {("empty", "filling"), ("filling", "full"), ("full", "draining"), ("draining", "empty")}


class PingPongBuffer:
    """The two-slot handoff of pipeline.py:67-149 (empty -> filling -> full ->
    draining -> empty), as the device ran it.

    On the B200 the handoff is two CUDA events per timestep: the model stream
    records "full" once the quantiser has written slot ``i % 2`` and the
    coder stream waits on it, encodes and records "empty", which the model
    stream waits on before it reuses the slot.  The kernels stamp each of
    those moments with the device clock into the executor's event tape
    (``fade_compress`` ``tape``: fill begins, table full, drain begins, drain
    done per step).  ``replay_tape`` feeds the recorded transitions through
    the reference's legality check in device-time order, so a ``trace``
    callback observes the schedule that actually ran -- including warm-up
    steps, whose uniform tables the warm-up kernel codes before the first
    model step.
    """

    def __init__(self, trace=None):
        self._states = ["empty", "empty"]
        self._trace = trace

    def _set(self, slot: int, new: str) -> None:
        old = self._states[slot]
        assert (old, new) in _LEGAL, f"illegal slot transition {old} -> {new}"
        self._states[slot] = new
        if self._trace is not None:
            self._trace((slot, old, new))

    def replay_tape(self, warm: int, tape) -> list:
        """Replay ``warm`` uniform-table steps, then the device tape
        ([steps, 5] int64 ns).  Returns the (t_ns, step, slot, new_state)
        events in the order they were applied."""
        events = []
        for i in range(warm):            # coded back to back by k_encode_warm
            for st in ("filling", "full", "draining", "empty"):
                events.append((0, i, i % 2, st))
        tape = np.asarray(tape, dtype=np.int64).reshape(-1, 5) if tape is not None else \
            np.zeros((0, 5), np.int64)
        timed = []
        for k, row in enumerate(tape):
            i = warm + k
            for st, t in zip(("filling", "full", "draining", "empty"), row[:4]):
                timed.append((int(t), i, i % 2, st))
        # device-time order; a tie keeps the protocol order of one step
        order = {"filling": 0, "full": 1, "draining": 2, "empty": 3}
        timed.sort(key=lambda e: (e[0], e[1], order[e[3]]))
        events += timed
        for _, _, slot, st in events:
            self._set(slot, st)
        return events


@dataclass
class CompressResult:
    streams: list
    cfg: ModelConfig
    partition: StreamPartition
    losses: list = field(default_factory=list)
    elapsed: float = 0.0
    metrics: list | None = None
    device: int | None = None     # CUDA device that ran the model (v2 shard fingerprint)


def _metrics(phase: str, first_step: int, losses, bytes_per_step: int, alpha=None,
             tape=None) -> list:
    """Per-step records of the --metrics tape (pipeline.py:162-185).

    Loss, router statistics (mean, min, max of alpha, model.py:197-199) and the
    clock all come from the device: ``elapsed_s`` is the %globaltimer time
    from the start of the first model step to the end of this one (event
    tape slot 4), so per-step timing is measured, not interpolated.
    """
    t = np.asarray(tape, dtype=np.int64).reshape(-1, 5) if tape is not None else None
    recs = []
    for k, loss in enumerate(losses):
        el = float(t[k, 4] - t[0, 0]) * 1e-9 if t is not None else 0.0
        rec = {"phase": phase, "step": first_step + k, "loss_nats": float(loss),
               "bits_per_byte": float(loss) / LN2, "elapsed_s": el,
               "kb_per_min": ((first_step + k + 1) * bytes_per_step / 1024.0)
               / max(el / 60.0, 1e-9)}
        if alpha is not None:
            rec.update(alpha_mean=float(alpha[k, 0]), alpha_min=float(alpha[k, 1]),
                       alpha_max=float(alpha[k, 2]))
        recs.append(rec)
    return recs


def _prepare(data: bytes, cfg: ModelConfig):
    cfg = cfg.shrink_to_fit(len(data))
    cfg.validate()
    part = StreamPartition.from_length(len(data), cfg.batch)
    mat = part.split(data)
    warm = min(cfg.ctx_len, part.stream_length)
    return cfg, part, mat, warm


def _raise_device(status: int, err: _native.FadeError, what: str):
    if status == 3:
        raise CorruptionError(int(err.stream), int(err.step), _native.last_error())
    if status == 4:
        raise ModelDivergenceError(int(err.step), _native.last_error())
    if status == 5:
        raise ValueError(f"row {int(err.stream)} does not sum to 1 within quantizer tolerance")
    raise RuntimeError(f"{what} failed (status {status}): {_native.last_error()}")


def _compress(data: bytes, cfg: ModelConfig, variant: str, pipelined: bool,
              collect_metrics: bool, trace=None, device=None) -> CompressResult:
    t0 = time.perf_counter()
    if not data:
        return CompressResult([], cfg, StreamPartition.from_length(0, cfg.batch))
    cfg, part, mat, warm = _prepare(data, cfg)
    steps = part.stream_length
    dev = default_device() if device is None else int(device)
    model = Predictor(cfg, variant, device=dev) if steps > warm else None
    if model is None:
        _native.require_device()
    lib = _native.lib()
    lengths = np.zeros(cfg.batch, dtype=np.int64)
    nsteps = steps - warm
    losses = np.zeros(max(nsteps, 1), dtype=np.float64)
    coder = ctypes.c_void_p()
    err = _native.FadeError()
    mat = np.ascontiguousarray(mat)
    routed = variant not in ("global_only", "local_only")   # alpha exists (model.py:146-151)
    alpha = np.zeros((max(nsteps, 1), 3), dtype=np.float64) if collect_metrics and routed else None
    want_tape = collect_metrics or trace is not None
    tape = np.zeros((max(nsteps, 1), 5), dtype=np.uint64) if want_tape else None
    st = lib.fade_compress(model.handle if model else None, dev, cfg.batch, mat.ctypes.data,
                           steps, warm, 0, 1 if pipelined else 0, lengths.ctypes.data,
                           losses.ctypes.data, alpha.ctypes.data if alpha is not None else None,
                           tape.ctypes.data if tape is not None else None,
                           ctypes.byref(coder), ctypes.byref(err))
    if st != 0:
        _raise_device(st, err, "fade_compress")
    try:
        payload = np.empty(int(lengths.sum()), dtype=np.uint8)
        _native.check(lib.fade_coder_fetch(coder, payload.ctypes.data, payload.size),
                      "fade_coder_fetch")
    finally:
        lib.fade_coder_destroy(coder)
    offs = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    streams = [payload[offs[k]:offs[k + 1]].tobytes() for k in range(cfg.batch)]
    loss_list = [float(x) for x in losses[:nsteps]] if nsteps > 0 else []
    elapsed = time.perf_counter() - t0
    tape_rows = tape[:nsteps].astype(np.int64) if tape is not None and nsteps > 0 else None
    if trace is not None:
        PingPongBuffer(trace).replay_tape(warm, tape_rows)
    metrics = (_metrics("compress", warm, loss_list, cfg.batch,
                        alpha if model is not None else None, tape_rows)
               if collect_metrics else None)
    return CompressResult(streams, cfg, part, loss_list, elapsed, metrics, dev)


def run_serial_compress(data: bytes, cfg: ModelConfig, variant: str = "full",
                        coder_delay: float = 0.0, collect_metrics: bool = False,
                        device: int | None = None) -> CompressResult:
    """predict -> quantise -> encode -> train per step, one CUDA stream (pipeline.py:197-226).

    ``coder_delay`` (the reference's latency injection) has no device analogue
    and is accepted for API compatibility only.  ``device``: the CUDA device
    to run on (default: ``model.default_device()``).
    """
    return _compress(data, cfg, variant, False, collect_metrics, device=device)


def run_pipelined_compress(data: bytes, cfg: ModelConfig, variant: str = "full",
                           coder_delay: float = 0.0, collect_metrics: bool = False,
                           trace=None, device: int | None = None) -> CompressResult:
    """CSPP: coder stream double-buffered against the model stream (pipeline.py:229-299).

    ``trace`` receives the (slot, old, new) transitions of the two-slot
    buffer in the order the device ran them (``PingPongBuffer.replay_tape``).
    """
    return _compress(data, cfg, variant, True, collect_metrics, trace, device)


def clamp_workers(workers: int, n_streams: int) -> int:
    """Largest worker count <= requested that divides the stream count (pipeline.py:302-307)."""
    w = max(1, min(int(workers), n_streams))
    while n_streams % w:
        w -= 1
    return w


def run_parallel_decompress(payload: np.ndarray, offsets: np.ndarray, lengths: np.ndarray,
                            cfg: ModelConfig, original_length: int, workers: int = 1,
                            decode_delay: float = 0.0, want_losses: bool = False,
                            collect_metrics: bool = False, device: int | None = None):
    """Decode every stream while replaying the encoder's updates (pipeline.py:310-396).

    One lane per stream replaces the reference's worker threads and their two
    barriers per step; ``workers`` is accepted and clamped for API parity.
    """
    if original_length == 0:
        return (b"", []) if want_losses else b""
    clamp_workers(workers, cfg.batch)
    part = StreamPartition.from_length(original_length, cfg.batch)
    steps = part.stream_length
    warm = min(cfg.ctx_len, steps)
    dev = default_device() if device is None else int(device)
    model = Predictor(cfg, device=dev) if steps > warm else None
    if model is None:
        _native.require_device()
    pay = np.asarray(payload, dtype=np.uint8)
    offsets = np.asarray(offsets, dtype=np.int64)
    lengths = np.ascontiguousarray(np.asarray(lengths, dtype=np.int64))
    # the device decoder takes streams back to back; regather if they are not
    std = np.concatenate([[0], np.cumsum(lengths)[:-1]]).astype(np.int64)
    if not np.array_equal(offsets, std) or pay.size != int(lengths.sum()):
        pay = np.concatenate([pay[o:o + n] for o, n in zip(offsets, lengths)]) \
            if len(lengths) else pay[:0]
    pay = np.ascontiguousarray(pay)
    out = np.zeros((cfg.batch, steps), dtype=np.uint8)
    nsteps = steps - warm
    losses = np.zeros(max(nsteps, 1), dtype=np.float64)
    alpha = np.zeros((max(nsteps, 1), 3), dtype=np.float64) if collect_metrics else None
    tape = np.zeros((max(nsteps, 1), 5), dtype=np.uint64) if collect_metrics else None
    err = _native.FadeError()
    st = _native.lib().fade_decompress(model.handle if model else None, dev, cfg.batch,
                                       pay.ctypes.data if pay.size else None, pay.size,
                                       lengths.ctypes.data, steps, warm, out.ctypes.data,
                                       losses.ctypes.data,
                                       alpha.ctypes.data if alpha is not None else None,
                                       tape.ctypes.data if tape is not None else None,
                                       ctypes.byref(err))
    if st != 0:
        _raise_device(st, err, "fade_decompress")
    data = part.join(out)
    loss_list = [float(x) for x in losses[:nsteps]] if nsteps > 0 else []
    if want_losses:
        return data, loss_list
    if collect_metrics:
        rows = tape[:nsteps].astype(np.int64) if nsteps > 0 else None
        return data, _metrics("decompress", warm, loss_list, cfg.batch,
                              alpha if model is not None else None, rows)
    return data


def throughput_report(n_bytes: int, compress_s: float, decompress_s: float) -> dict:
    """KB/min; the total is the harmonic 2*size over the summed time (pipeline.py:399-411)."""
    kb = n_bytes / 1024.0
    return {
        "n_bytes": n_bytes,
        "compress_s": compress_s,
        "decompress_s": decompress_s,
        "compress_kb_min": kb / max(compress_s / 60.0, 1e-12),
        "decompress_kb_min": kb / max(decompress_s / 60.0, 1e-12),
        "total_kb_min": 2.0 * kb / max((compress_s + decompress_s) / 60.0, 1e-12),
    }
