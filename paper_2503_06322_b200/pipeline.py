"""Overlapped host<->device reduction pipeline (paper §V: HDEM, Fig. 7, Algorithm 4).

The reference package names this subsystem (hpdr/pipeline/__init__.py:4-19) but ships only
its chunk-size models (hpdr/pipeline/models.py); the runner is rebuilt here on CUDA streams in
libhpdr_b200.so (csrc/pipeline.cu).  Each dim-0 chunk becomes a reference-identical MGARD blob
compressed with the global value range, stored in an HPDR container (container.py).

Host-side scheduling (this module):
  ThroughputModel / TransportModel / next_chunk_size / fit_throughput_model  -- Φ, Θ and the
      Algorithm-4 rule (models.py:22-120), restated
  adaptive_schedule  -- the chunk sequence Algorithm 4 produces for a field
  overlap_ratio      -- SPEC.md's overlap metric over a pipeline trace
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, dims_arg, lib
from .errors import ValidationError

FIT_CUTOFF = 0.1        # models.py:17
SATURATION_TOL = 0.05   # models.py:19


# ----------------------------------------------------------------------------- models
@dataclass
class ThroughputModel:
    """Φ(C): linear ramp below c_threshold, plateau gamma above (bytes/s)."""

    alpha: float
    beta_slope: float
    gamma: float
    c_threshold: float
    f: float = FIT_CUTOFF

    def phi(self, chunk_bytes: float) -> float:
        c = float(chunk_bytes)
        v = self.gamma if c >= self.c_threshold else self.alpha * c + self.beta_slope
        if v <= 0:
            raise ValidationError(f"throughput model non-positive at {chunk_bytes}")
        return v

    @classmethod
    def saturated(cls, gamma: float) -> "ThroughputModel":
        return cls(0.0, float(gamma), float(gamma), 0.0)


@dataclass
class TransportModel:
    """Θ(t) = t / beta_copy, beta_copy in seconds per byte (EMA-updated from observed copies)."""

    beta_copy: float
    ema_weight: float = 0.25

    def __post_init__(self):
        if self.beta_copy <= 0:
            raise ValidationError("beta_copy must be > 0")

    def theta(self, seconds: float) -> float:
        return float(seconds) / self.beta_copy

    def observe(self, nbytes: int, seconds: float):
        if nbytes > 0 and seconds > 0:
            self.beta_copy += self.ema_weight * (seconds / nbytes - self.beta_copy)


def next_chunk_size(c_curr: int, model: ThroughputModel, transport: TransportModel, c_limit: int,
                    size_rest: int, slab_bytes: int = 1) -> int:
    """Algorithm 4 line 17: min(Θ(C/Φ(C)), C_limit, rest), floored to whole slabs, never 0."""
    if size_rest <= 0:
        return 0
    if c_curr <= 0:
        raise ValidationError("c_curr must be > 0")
    want = min(transport.theta(c_curr / model.phi(c_curr)), float(c_limit), float(size_rest))
    slabs = max(1, int(want // slab_bytes))
    return int(min(slabs * slab_bytes, size_rest))


def fit_throughput_model(samples, f: float = FIT_CUTOFF) -> ThroughputModel:
    """Plateau from the largest profiled chunk; least-squares ramp over the points below the
    plateau down to the first one under f * plateau (§V-C)."""
    pts = sorted((float(c), float(p)) for c, p in samples)
    if len(pts) < 3:
        raise ValidationError("need at least 3 profile samples")
    if len({c for c, _ in pts}) == 1:
        raise ValidationError("degenerate profile: all sizes equal")
    gamma = pts[-1][1]
    if gamma <= 0:
        raise ValidationError("non-positive saturated throughput")
    ramp = []
    for c, p in reversed(pts[:-1]):
        if p >= gamma * (1.0 - SATURATION_TOL):
            continue
        if p < f * gamma:
            break
        ramp.append((c, p))
    smallest = pts[0][0]
    if len(ramp) >= 2:
        a, b = np.polyfit([c for c, _ in ramp], [p for _, p in ramp], 1)
        a, b = float(a), float(b)
        if a > 0:
            return ThroughputModel(a, b, gamma, (gamma - b) / a, f)
    return ThroughputModel(0.0, gamma, gamma, smallest, f)


def adaptive_schedule(n0: int, plane_bytes: int, model: ThroughputModel, transport: TransportModel,
                      c_init: int = 16 << 20, c_limit: int | None = None) -> list:
    """Chunk plane counts Algorithm 4 produces for a field of n0 planes."""
    total = n0 * plane_bytes
    c_limit = c_limit or total
    planes = []
    rest = total
    c = min(max(plane_bytes, (c_init // plane_bytes) * plane_bytes), rest)
    while rest > 0:
        c = min(c, rest)
        planes.append(max(1, c // plane_bytes))
        rest -= planes[-1] * plane_bytes
        if rest > 0:
            c = next_chunk_size(planes[-1] * plane_bytes, model, transport, c_limit, rest, plane_bytes)
    return planes


def _host_view(arr) -> np.ndarray:
    """A numpy view (or, for a CUDA tensor, a host copy) of an input array."""
    if hasattr(arr, "numpy"):
        return arr.cpu().numpy() if getattr(arr, "is_cuda", False) else arr.numpy()
    if hasattr(arr, "values") and hasattr(arr, "dims"):   # TensorData
        return np.asarray(arr.values)
    return np.asarray(arr)


def profile_models(arr, eb_rel: float, sizes_mb=(16, 32, 64, 128, 256), *, device: int | None = None,
                   reps: int = 2):
    """Fit Φ and Θ on this device (§V-C): Φ(C) = compress throughput of a device-resident
    C-byte slab of `arr` (no copies), Θ from a pinned host-to-device copy of the largest slab.
    Returns (ThroughputModel, TransportModel, samples)."""
    import time

    from .mgard import _as_input, mgard_compress

    addr, dims, code, keep = _as_input(arr)
    a = _host_view(arr)
    plane_bytes = a[0].nbytes
    ctx = _lib.default_context(device, arr if getattr(arr, 'is_cuda', False) else None)
    samples = []
    import torch

    dev = torch.device("cuda", ctx.device if hasattr(ctx, "device") else 0)
    plane_counts = [max(1, min(a.shape[0], int(mb * (1 << 20)) // plane_bytes)) for mb in sizes_mb]
    if len(set(plane_counts)) < 3:   # a field smaller than the sweep: profile fractions of it
        plane_counts = sorted({max(1, a.shape[0] * k // 8) for k in (1, 2, 4, 8)})
    for planes in plane_counts:
        slab = torch.from_numpy(np.ascontiguousarray(a[:planes])).to(dev)
        vr = (float(a.min()), float(a.max()))
        sink = torch.empty(slab.numel() * slab.element_size() * 2 + (8 << 20), dtype=torch.uint8, device=dev)
        mgard_compress(slab, eb_rel, value_range=vr, device=device, out=sink)   # warm (tables, buffers)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for _ in range(reps):
            mgard_compress(slab, eb_rel, value_range=vr, device=device, out=sink)   # blob stays on the device
        torch.cuda.synchronize(dev)
        dt = (time.perf_counter() - t0) / reps
        samples.append((slab.numel() * slab.element_size(), slab.numel() * slab.element_size() / dt))
    big = torch.from_numpy(np.ascontiguousarray(a[: max(1, min(a.shape[0], (max(sizes_mb) << 20) // plane_bytes))]))
    pin = big.pin_memory()
    d = torch.empty_like(pin, device=dev)
    d.copy_(pin, non_blocking=True)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    d.copy_(pin, non_blocking=True)
    torch.cuda.synchronize(dev)
    beta = (time.perf_counter() - t0) / pin.nbytes
    del keep
    return fit_throughput_model(samples), TransportModel(beta), samples


def compress_adaptive(arr, eb_rel: float, dict_size: int = 4096, value_range=None, *, models=None,
                      c_init: int = 16 << 20, c_limit: int = 1 << 30, device: int | None = None, out=None,
                      trace: bool = False):
    """Algorithm 4 end to end: chunk sizes from the fitted Φ / Θ (profile_models, or `models`),
    then the streams pipeline over that schedule.  Returns what compress_pipelined returns."""
    a = _host_view(arr)
    if models is None:
        phi, theta, _ = profile_models(arr, eb_rel, device=device)
    else:
        phi, theta = models
    sched = adaptive_schedule(a.shape[0], a[0].nbytes, phi, theta, c_init=c_init, c_limit=c_limit)
    return compress_pipelined(arr, eb_rel, dict_size, value_range, chunks=sched, device=device, out=out,
                              trace=trace)


def overlap_ratio(trace: np.ndarray) -> float:
    """SPEC.md overlap: time during which a copy (H2D or D2H) overlaps any compute / total copy time.
    trace: (K, 6) = H2D start/end, compute start/end, D2H start/end (ms)."""
    t = np.asarray(trace, dtype=np.float64).reshape(-1, 6)
    if t.size == 0:
        return 0.0
    comp = sorted((a, b) for a, b in t[:, 2:4])
    copies = [(a, b) for a, b in t[:, 0:2]] + [(a, b) for a, b in t[:, 4:6]]
    total = sum(max(0.0, b - a) for a, b in copies)
    if total <= 0:
        return 0.0
    ov = 0.0
    for a, b in copies:
        for ca, cb in comp:
            ov += max(0.0, min(b, cb) - max(a, ca))
    return min(1.0, ov / total)


TRACE_COLUMNS = ("task_kind", "chunk_id", "queue", "start_ns", "end_ns")
QUEUES = 3   # chunks go round-robin to the three queues of Fig. 7 (pipeline.cu)


def trace_rows(trace: np.ndarray, queues: int = QUEUES):
    """A runner trace (K, 6) in ms as SPEC.md's export rows (task_kind, chunk_id, queue, start_ns,
    end_ns): one H2D, COMPUTE and D2H task per chunk, times relative to the earliest start."""
    t = np.asarray(trace, dtype=np.float64).reshape(-1, 6)
    if t.size == 0:
        return []
    t0 = float(t.min())
    rows = []
    for k, r in enumerate(t):
        for kind, (a, b) in zip(("H2D", "COMPUTE", "D2H"), ((r[0], r[1]), (r[2], r[3]), (r[4], r[5]))):
            rows.append((kind, k, k % queues, int(round((a - t0) * 1e6)), int(round((b - t0) * 1e6))))
    rows.sort(key=lambda x: (x[3], x[1]))
    return rows


def write_trace_csv(trace: np.ndarray, f, queues: int = QUEUES) -> int:
    """SPEC.md trace export (External Interfaces): CSV with columns task_kind, chunk_id, queue,
    start_ns, end_ns.  ``f`` is a path or a text file object; returns the number of task rows."""
    import csv

    rows = trace_rows(trace, queues)
    own = isinstance(f, (str, bytes, os.PathLike))
    fh = open(f, "w", newline="") if own else f
    try:
        w = csv.writer(fh)
        w.writerow(TRACE_COLUMNS)
        w.writerows(rows)
    finally:
        if own:
            fh.close()
    return len(rows)


# ----------------------------------------------------------------------------- runner
def compress_pipelined(arr, eb_rel: float, dict_size: int = 4096, value_range=None, *, chunk_planes: int = 0,
                       chunks=None, device: int | None = None, out=None, trace: bool = False):
    """Chunked compress through the streams pipeline -> HPDR container bytes.

    ``chunks`` (plane counts summing to dim 0) overrides the fixed ``chunk_planes``.
    With ``trace`` returns (bytes, trace array of shape (K, 6) in ms).
    """
    from .mgard import _as_input, _dims_ok

    addr, dims, code, keep = _as_input(arr)
    dims = _dims_ok(dims)
    ctx = _lib.default_context(device, arr if getattr(arr, "is_cuda", False) else out)
    has = value_range is not None
    r0, r1 = (float(value_range[0]), float(value_range[1])) if has else (0.0, 0.0)
    lst = None if chunks is None else np.ascontiguousarray(chunks, dtype=np.uint64)
    k = len(lst) if lst is not None else -(-dims[0] // chunk_planes) if chunk_planes else 0
    nbytes = int(np.prod(dims)) * (4 if code == 0 else 8)
    cap = nbytes + (1 << 20) if out is None else int(out.nbytes)
    buf = _lib.pinned_scratch(cap) if out is None else out   # reused pinned scratch, then one bytes copy
    tr = np.zeros(6 * max(k, 1) + 6 * 4096, np.float64) if trace else None
    n = C.c_uint64()

    def run(b):
        return lib().hpdr_pipeline_compress(
            ctx.handle, C.c_void_p(addr), code, len(dims), dims_arg(dims), float(eb_rel), int(dict_size), int(has),
            r0, r1, int(chunk_planes), C.c_void_p(lst.ctypes.data) if lst is not None else None,
            0 if lst is None else len(lst), C.c_void_p(_lib.ptr(b)), int(b.nbytes), C.byref(n),
            C.c_void_p(tr.ctypes.data) if tr is not None else None)

    rc = run(buf)
    if rc == _lib.BUFFER and out is None:   # incompressible data: worst-case bound
        buf = np.empty(nbytes * 6 + (8 << 20), np.uint8)
        rc = run(buf)
    check(rc)
    del keep
    data = _lib.bytes_from(buf, n.value) if out is None else int(n.value)
    if not trace:
        return data
    from .container import read_container

    h, _ = read_container(buf[: n.value] if out is None else out[: n.value])
    return data, tr[: 6 * len(h.chunks)].reshape(-1, 6)


def decompress_pipelined(data, *, device: int | None = None, out=None, trace: bool = False):
    """Decompress an HPDR container through the streams pipeline."""
    from .container import read_container
    from .tensor import DTYPE_FROM_CODE

    buf = np.frombuffer(memoryview(data), np.uint8)
    h, _ = read_container(buf)
    res = np.empty(h.dims, DTYPE_FROM_CODE[h.dtype].np_dtype) if out is None else out
    tr = np.zeros(6 * max(1, len(h.chunks)), np.float64) if trace else None
    ctx = _lib.default_context(device, data if getattr(data, "is_cuda", False) else out)
    check(lib().hpdr_pipeline_decompress(ctx.handle, C.c_void_p(buf.ctypes.data), buf.size,
                                         C.c_void_p(_lib.ptr(res)), int(res.nbytes),
                                         C.c_void_p(tr.ctypes.data) if tr is not None else None))
    if trace:
        return res, tr[: 6 * len(h.chunks)].reshape(-1, 6)
    return res
