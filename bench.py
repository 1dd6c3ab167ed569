#!/usr/bin/env python
"""Benchmark of the B200 MGARD reduction path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

One step = one mgard_compress of the workload (BASELINE configs[1] by default: a 513^3 fp32
smooth+noise field, relative L-inf bound 1e-4), the reference's drop-in call.  Rank 0 prints
one JSON line:
  value    compress GB/s with the input resident in HBM and the blob left on the device
           (whole job: input bytes of all ranks / max-over-ranks time)
  e2e      the same call through the C ABI with pinned HOST buffers: H2D of the field, kernels,
           D2H of the blob, every step
  decompress   the mirror direction (kernel-only and end-to-end)
  roofline the dominant kernel's algorithmic bytes / CUDA-event duration vs measured HBM peak
  cpu_baseline the C parity oracle (a port of the reference algorithm) on this host's cores
Multi-GPU: every rank reduces its own block (weak scaling); only the global min/max
(2 doubles, all-reduce) and the blob sizes (all-gather) cross ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "compress/decompress GB/s end-to-end (H2D+kernel+D2H) at 1/2/4/8 B200 vs CPU ref"

CONFIGS = {
    "c2": dict(workload="configs[1]: 3D fp32 513^3 smooth+noise field, rel L-inf 1e-4", shape=(513, 513, 513),
               dtype="f32", field="smooth", eb=1e-4),
    "c1": dict(workload="configs[0]: 3D fp32 129^3 GRF, abs L-inf 1e-3", shape=(129, 129, 129), dtype="f32",
               field="grf", eb=1e-3, value_range=(0.0, 1.0)),
    "c3": dict(workload="configs[2]: NYX-like 512^3 fp32 temperature, rel 1e-3", shape=(512, 512, 512), dtype="f32",
               field="temperature", eb=1e-3),
    "c4": dict(workload="configs[3]: 3D fp64 128x1024x1024 slab per rank of a 1024^3 field, global range, rel 1e-4",
               shape=(128, 1024, 1024), dtype="f64", field="smooth", eb=1e-4),
    "c5": dict(workload="configs[4]: 1024^3 fp32 timestep", shape=(1024, 1024, 1024), dtype="f32", field="smooth",
               eb=1e-2),
}


def make_field(cfg, seed):
    from paper_2503_06322_b200 import synthetic as S

    dt = np.float32 if cfg["dtype"] == "f32" else np.float64
    if cfg["field"] == "smooth":
        return S.smooth_noise(cfg["shape"], seed=seed, dtype=dt)
    if cfg["field"] == "grf":
        return S.grf(cfg["shape"], m=8, seed=seed, dtype=dt)
    return S.nyx_like(cfg["shape"], cfg["field"], seed=seed, dtype=dt)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(kernel):
    """DRAM bytes (read + write) of one launch of `kernel` from this round's committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        return t.get(kernel)
    except Exception:
        return None


def pcie_roofline(dev, mib=256, reps=3):
    """Pinned H2D / D2H bandwidth on this box (the end-to-end roofline denominators), CUDA events."""
    import torch

    n = mib << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    out = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        for _ in range(2):
            fn()
        torch.cuda.synchronize(dev)
        best = 0.0
        for _trial in range(3):   # best of 3: a one-off stall must not lower the roofline
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            e1.synchronize()
            best = max(best, n * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        out[name] = best
    return out


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            self.p.wait()

    def summary(self):
        self.f.flush()
        self.f.seek(0)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() in ("active", "1", "yes"):
                    reasons.add(n)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_oracle_time(cfg, a, budget_s=20.0):
    """Time the C port of the reference algorithm on this host's cores, on a bounded slab sample."""
    from oracle import oracle as O

    threads = os.cpu_count() or 1
    O.set_threads(threads)
    vr = cfg.get("value_range")
    planes = min(a.shape[0], 33)
    t0 = time.perf_counter()
    O.mgard_compress(np.ascontiguousarray(a[:planes]), cfg["eb"], value_range=vr)
    t_probe = time.perf_counter() - t0
    per_plane = t_probe / planes
    planes = int(max(9, min(a.shape[0], budget_s / 3.0 / max(per_plane, 1e-9))))
    sample = np.ascontiguousarray(a[:planes])
    reps, tc, td = 0, 0.0, 0.0
    blob = None
    while reps < 3 and (tc + td) < budget_s:
        t0 = time.perf_counter()
        blob = O.mgard_compress(sample, cfg["eb"], value_range=vr)
        t1 = time.perf_counter()
        O.mgard_decompress(blob)
        t2 = time.perf_counter()
        tc += t1 - t0
        td += t2 - t1
        reps += 1
    nb = sample.nbytes * reps
    return dict(compress_gbs=nb / tc / 1e9, decompress_gbs=nb / td / 1e9, cores=threads,
                sample=f"first {planes} planes of the workload ({sample.nbytes / 1e6:.0f} MB) x {reps}, "
                       f"C oracle (port of hpdr/mgard), OpenMP {threads} threads")


def cpu_zfp_time(a, rate, budget_s=6.0):
    """The fixed-rate coder's C port (oracle/zfp_oracle.c) on this host's cores, whole field."""
    from oracle import oracle as O

    threads = os.cpu_count() or 1
    O.set_threads(threads)
    reps, tc, td = 0, 0.0, 0.0
    while reps < 3 and (tc + td) < budget_s:
        t0 = time.perf_counter()
        blob = O.zfp_compress(a, rate)
        t1 = time.perf_counter()
        O.zfp_decompress(blob)
        t2 = time.perf_counter()
        tc += t1 - t0
        td += t2 - t1
        reps += 1
    nb = a.nbytes * reps
    return dict(compress_gbs=nb / tc / 1e9, decompress_gbs=nb / td / 1e9, cores=threads,
                sample=f"whole field ({a.nbytes / 1e6:.0f} MB) x {reps}, C oracle (port of hpdr/zfp.py), "
                       f"OpenMP {threads} threads")


def run_reference(args, cfg, rank):
    if rank != 0:
        return
    a = make_field(cfg, seed=0)
    from oracle import oracle as O

    threads = os.cpu_count() or 1
    O.set_threads(threads)
    vr = cfg.get("value_range")
    planes = min(a.shape[0], 33)
    t0 = time.perf_counter()
    O.mgard_compress(np.ascontiguousarray(a[:planes]), cfg["eb"], value_range=vr)
    per_plane = (time.perf_counter() - t0) / planes
    # bound the whole --steps K --warmup W run to ~2 minutes of CPU work
    budget_step = 120.0 / max(1, args.steps + args.warmup)
    planes = int(max(9, min(a.shape[0], budget_step / max(per_plane, 1e-9))))
    sample = np.ascontiguousarray(a[:planes])
    for _ in range(args.warmup):
        O.mgard_compress(sample, cfg["eb"], value_range=vr)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.mgard_compress(sample, cfg["eb"], value_range=vr)
    dt = time.perf_counter() - t0
    v = sample.nbytes * args.steps / dt / 1e9
    line = {"metric": METRIC, "impl": "reference", "value": v, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": cfg["workload"], "shape": list(cfg["shape"]),
                                            "eb_rel": cfg["eb"], "direction": "compress"},
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": threads, "kind": "port",
                             "sample": f"first {planes} of {a.shape[0]} planes per step, C oracle port of "
                                       f"hpdr/mgard (OpenMP {threads} threads)"},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--zfp-rate", type=int, default=16, help="bits/value of the fixed-rate leg (0: skip)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, cfg, rank)
        return

    import torch
    import torch.distributed as dist

    import paper_2503_06322_b200 as P
    from paper_2503_06322_b200 import _lib

    # HPDR_BENCH_SAME_GPU=1 (testing the multi-rank path on a 1-GPU box): every rank on GPU 0,
    # metadata collectives over gloo
    if os.environ.get("HPDR_BENCH_SAME_GPU") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if os.environ.get("HPDR_BENCH_SAME_GPU") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    a = make_field(cfg, seed=rank)                      # this rank's block (weak scaling)
    nbytes = a.nbytes
    ctx = _lib.default_context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    code = 0 if a.dtype == np.float32 else 1
    d_in = torch.from_numpy(a).to(dev)                 # HBM-resident input for the kernel-only number
    h_in = torch.from_numpy(a).pin_memory()            # pinned host input for e2e

    def global_range(ptr):
        if world == 1 and cfg.get("value_range") is None:
            return None
        if cfg.get("value_range") is not None:
            return cfg["value_range"]
        lo, hi = _lib.minmax(ctx, ptr, code, a.size)
        t = torch.tensor([-lo, hi], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)     # 16 bytes: the only data-path exchange
        return (-float(t[0]), float(t[1]))

    def compress_dev():
        vr = global_range(d_in.data_ptr())
        return P.mgard_compress(d_in, cfg["eb"], value_range=vr, out=dummy_out)

    # kernel-only output stays on the device: compress into a device buffer
    blob_ref = P.mgard_compress(d_in, cfg["eb"], value_range=global_range(d_in.data_ptr()))
    blob_len = len(blob_ref)
    dummy_out = torch.empty(blob_len + (1 << 20), dtype=torch.uint8, device=dev)
    h_blob = torch.empty(blob_len + (1 << 20), dtype=torch.uint8).pin_memory()

    # End to end with N > 1 ranks the global range (2 doubles, all-reduced once before timing) is
    # passed as the value range, i.e. an absolute bound: the blobs are identical to the relative-
    # mode ones, and the field is not read twice per step.
    vr_e2e = global_range(d_in.data_ptr()) if world > 1 else cfg.get("value_range")

    def compress_e2e():
        n = P.mgard_compress(h_in, cfg["eb"], value_range=vr_e2e, out=h_blob)
        return n

    d_out = torch.empty(a.shape, dtype=d_in.dtype, device=dev)
    h_out = torch.empty(a.shape, dtype=d_in.dtype).pin_memory()
    h_blob_in = torch.from_numpy(np.frombuffer(blob_ref, np.uint8).copy()).pin_memory()
    blob_view = h_blob_in.numpy()

    d_blob = torch.from_numpy(np.frombuffer(blob_ref, np.uint8).copy()).to(dev)   # device-resident blob

    def decompress_dev():
        P.mgard_decompress(d_blob, out=d_out)

    def decompress_e2e():
        P.mgard_decompress(blob_view, out=h_out)

    # inputs smaller than the 126 MB L2: a 256 MB buffer written between timed steps
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev) if nbytes < (126 << 20) else None

    def timed(fn, steps, prof=False, clocks=None):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize(dev)
        barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        _lib.launch_count(reset=True)
        if prof:
            _lib.prof_enable(True)
        if flush is None:   # inputs larger than L2: one timed region over all steps
            e0.record(stream)
            for _ in range(steps):
                fn()
            e1.record(stream)
            e1.synchronize()
            total = e0.elapsed_time(e1)
        else:               # inputs smaller than L2: each step timed alone, L2 flushed in between
            total = 0.0
            for _ in range(steps):
                flush.add_(1)
                torch.cuda.synchronize(dev)
                e0.record(stream)
                fn()
                e1.record(stream)
                e1.synchronize()
                total += e0.elapsed_time(e1)
        torch.cuda.synchronize(dev)
        launches = _lib.launch_count()
        kern = _lib.prof_read() if prof else None
        if prof:
            _lib.prof_enable(False)
        barrier()
        ms = max_over_ranks(total)
        return ms / steps, launches, kern

    # M2: the paper's chunked streams pipeline (HPDR container of per-chunk reference blobs).
    # Streaming use takes an absolute bound (value range fixed up front), as for a timestep stream.
    from paper_2503_06322_b200 import pipeline as PL

    # relative mode as configured: the runner decomposes chunks as they stream in and quantizes
    # them once the global range is known (value_range only when the config fixes one)
    vr_abs = cfg.get("value_range") if world == 1 else vr_e2e
    pipe_out = torch.empty(nbytes + (64 << 20), dtype=torch.uint8).pin_memory().numpy()
    pipe_len = PL.compress_pipelined(h_in, cfg["eb"], value_range=vr_abs, out=pipe_out)
    pipe_in = torch.from_numpy(pipe_out[:pipe_len].copy()).pin_memory().numpy()
    h_out2 = torch.empty(a.shape, dtype=d_in.dtype).pin_memory().numpy()

    def compress_pipe():
        PL.compress_pipelined(h_in, cfg["eb"], value_range=vr_abs, out=pipe_out)

    # the same pipeline with the range known up front (a timestep stream with an absolute bound)
    vr_known = vr_abs or (float(a.min()), float(a.max()))

    def compress_pipe_abs():
        PL.compress_pipelined(h_in, cfg["eb"], value_range=vr_known, out=pipe_out)

    # Algorithm 4: chunk sizes from Φ (device-profiled) and Θ (pinned copy) -- a one-time
    # calibration per field shape, outside the timed region
    models = PL.profile_models(h_in, cfg["eb"])[:2]
    sched = PL.adaptive_schedule(a.shape[0], a[0].nbytes, *models, c_init=16 << 20, c_limit=1 << 30)

    def compress_pipe_adaptive():
        PL.compress_pipelined(h_in, cfg["eb"], value_range=vr_known, chunks=sched, out=pipe_out)

    def decompress_pipe():
        PL.decompress_pipelined(pipe_in, out=h_out2)

    # fixed-rate block coder (hpdr/zfp.py) on the same field
    from paper_2503_06322_b200 import zfp as ZF

    zrate = args.zfp_rate if a.ndim <= 3 else 0
    if zrate:
        z_len = ZF.compressed_size(a.shape, P.DType.F32 if code == 0 else P.DType.F64, zrate)
        z_dev = torch.empty(z_len, dtype=torch.uint8, device=dev)
        z_host = torch.empty(z_len, dtype=torch.uint8).pin_memory()
        ZF.zfp_compress(d_in, zrate, out=z_dev)
        z_blob = bytes(z_dev.cpu().numpy())
        z_host_in = torch.from_numpy(np.frombuffer(z_blob, np.uint8).copy()).pin_memory()

        def zfp_c_dev():
            ZF.zfp_compress(d_in, zrate, out=z_dev)

        def zfp_d_dev():
            ZF.zfp_decompress(z_dev, out=d_out)

        def zfp_c_e2e():
            ZF.zfp_compress(h_in, zrate, out=z_host)

        def zfp_d_e2e():
            ZF.zfp_decompress(z_host_in, out=h_out)

        # the fixed-rate reducer through the streams pipeline (HPDR container, pipeline id 1)
        zp_len = len(ZF.compress_pipelined(h_in, zrate))
        zp_out = torch.empty(zp_len, dtype=torch.uint8).pin_memory().numpy()
        ZF.compress_pipelined(h_in, zrate, out=zp_out)
        zp_in = torch.from_numpy(zp_out.copy()).pin_memory().numpy()
        zp_dec = torch.empty(a.shape, dtype=d_in.dtype).pin_memory().numpy()

        def zfp_pc():
            ZF.compress_pipelined(h_in, zrate, out=zp_out)

        def zfp_pd():
            PL.decompress_pipelined(zp_in, out=zp_dec)

    # the drop-in API exactly as a reference user calls it: numpy array in, Python bytes out (and back),
    # i.e. pageable host memory on both sides (staged through the library's pinned rings)
    blob_np = P.mgard_compress(a, cfg["eb"], value_range=vr_e2e)

    def pageable_c():
        P.mgard_compress(a, cfg["eb"], value_range=vr_e2e)

    def pageable_d():
        P.mgard_decompress(blob_np)

    K = args.steps
    pcie = pcie_roofline(dev)
    with ClockSampler(local) as clk:
        c_ms, launches, kern = timed(compress_dev, K, prof=True)
        e_ms, _, _ = timed(compress_e2e, K)
        d_ms, _, dkern = timed(decompress_dev, K, prof=True)
        de_ms, _, _ = timed(decompress_e2e, K)
        pc_ms, _, _ = timed(compress_pipe, K)
        pd_ms, _, _ = timed(decompress_pipe, K)
        pa_ms, _, _ = timed(compress_pipe_abs, K)
        pad_ms, _, _ = timed(compress_pipe_adaptive, K)
        pg_c_ms, _, _ = timed(pageable_c, K)
        pg_d_ms, _, _ = timed(pageable_d, K)
        if zrate:
            zc_ms, zc_l, zkern = timed(zfp_c_dev, K, prof=True)
            zd_ms, zd_l, zdkern = timed(zfp_d_dev, K, prof=True)
            zce_ms, _, _ = timed(zfp_c_e2e, K)
            zde_ms, _, _ = timed(zfp_d_e2e, K)
            zpc_ms, _, _ = timed(zfp_pc, K)
            zpd_ms, _, _ = timed(zfp_pd, K)
    clocks = clk.summary()
    _, ptr_c = PL.compress_pipelined(h_in, cfg["eb"], value_range=vr_abs, out=pipe_out, trace=True)
    _, ptr_d = PL.decompress_pipelined(pipe_in, out=h_out2, trace=True)
    vr_chk = vr_abs or (float(a.min()), float(a.max()))
    assert np.max(np.abs(h_out2.astype(np.float64) - a)) <= cfg["eb"] * (vr_chk[1] - vr_chk[0])

    # correctness guard on the measured outputs
    assert bytes(h_blob[:blob_len].numpy()) == blob_ref, "e2e blob differs from the device-path blob"
    out_np = h_out.numpy()
    rng_ = float(a.max()) - float(a.min()) if cfg.get("value_range") is None else \
        cfg["value_range"][1] - cfg["value_range"][0]
    max_err = float(np.max(np.abs(out_np.astype(np.float64) - a.astype(np.float64))))

    sizes = [blob_len]
    if world > 1:
        t = torch.tensor([blob_len], dtype=torch.int64, device=dev)
        g = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(g, t)                          # compressed-size metadata exchange
        sizes = [int(x.item()) for x in g]
    total_in = nbytes * world
    gbs = lambda ms: total_in / (ms * 1e-3) / 1e9  # noqa: E731

    hbm, peak_kind = measured_peaks()
    # dominant kernel of the kernel-only step (largest share of device time); its finest-level
    # launch carries the roofline (the coarser launches of the same kernel are a separate name)
    dname, (dl, dms, dbytes, dmax) = max(kern.items(), key=lambda kv: kv[1][1])
    achieved = dbytes / (dms * 1e-3) / 1e9
    traffic = ncu_traffic(dname)
    roofline = {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic, "algorithmic_bytes": dbytes / max(dl, 1),
                "launch_ms": dms / max(dl, 1), "peak_kind": peak_kind, "share_of_step": dms / (c_ms * K),
                "launches_per_step": dl / K,
                "traffic_source": "profiles/ncu_traffic.json (ncu --set full, dram__bytes_read+write)"}
    # end-to-end roofline: the copies alone at the measured pinned PCIe rates
    t_c = max(nbytes / (pcie["h2d"] * 1e9), blob_len / (pcie["d2h"] * 1e9))
    t_d = max(blob_len / (pcie["h2d"] * 1e9), nbytes / (pcie["d2h"] * 1e9))
    t_pc = max(nbytes / (pcie["h2d"] * 1e9), pipe_len / (pcie["d2h"] * 1e9))
    t_pd = max(pipe_len / (pcie["h2d"] * 1e9), nbytes / (pcie["d2h"] * 1e9))

    line = {
        "metric": METRIC, "value": gbs(c_ms), "unit": "GB/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": c_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["workload"], "shape": list(cfg["shape"]), "input_dtype": cfg["dtype"],
                   "eb_rel": cfg["eb"], "direction": "compress", "l2": "inputs larger than L2 (no flush needed)"
                   if nbytes > 126e6 else "inputs smaller than L2: 256 MB buffer written between separately timed steps",
                   "parallelism": f"block-partitioned x{world} (global range all-reduce only)",
                   "mode": "M1: mgard_compress drop-in, one reference-identical blob per rank"},
        "e2e": {"value": gbs(e_ms), "unit": "GB/s", "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": blob_len,
                "ms_per_step": e_ms, "memory": "pinned host in/out",
                "pcie_roofline_frac": t_c / (e_ms * 1e-3)},
        "decompress": {"value": gbs(d_ms), "ms_per_step": d_ms,
                       "e2e": {"value": gbs(de_ms), "unit": "GB/s", "h2d_bytes_per_step": blob_len,
                               "d2h_bytes_per_step": nbytes, "ms_per_step": de_ms,
                               "pcie_roofline_frac": t_d / (de_ms * 1e-3)}},
        "pipeline": {"mode": "M2 streams pipeline (HPDR container of per-chunk reference blobs), 64 MB chunks, "
                             "3 queues, relative bound with the global range (chunks decomposed on arrival, "
                             "quantized once the range is known)" if vr_abs is None else
                             "M2 streams pipeline, 64 MB chunks, 3 queues, value_range given",
                     "compress_e2e_gbs": gbs(pc_ms), "decompress_e2e_gbs": gbs(pd_ms),
                     "compress_ms": pc_ms, "decompress_ms": pd_ms, "cr": nbytes / pipe_len,
                     "compress_pcie_roofline_frac": t_pc / (pc_ms * 1e-3),
                     "decompress_pcie_roofline_frac": t_pd / (pd_ms * 1e-3),
                     "compress_abs_e2e_gbs": gbs(pa_ms), "compress_abs_ms": pa_ms,
                     "compress_abs_pcie_roofline_frac": t_pc / (pa_ms * 1e-3),
                     "compress_adaptive_abs_e2e_gbs": gbs(pad_ms), "compress_adaptive_abs_ms": pad_ms,
                     "compress_adaptive_abs_pcie_roofline_frac": t_pc / (pad_ms * 1e-3),
                     "adaptive_chunks_planes": [int(x) for x in sched],
                     "chunks": int(ptr_c.shape[0]), "overlap_compress": PL.overlap_ratio(ptr_c),
                     "overlap_decompress": PL.overlap_ratio(ptr_d)},
        "pageable": {"mode": "drop-in API with a numpy array in / Python bytes out (pageable host memory)",
                     "compress_e2e_gbs": gbs(pg_c_ms), "decompress_e2e_gbs": gbs(pg_d_ms),
                     "compress_ms": pg_c_ms, "decompress_ms": pg_d_ms},
        "pcie": {"h2d_gbs": pcie["h2d"], "d2h_gbs": pcie["d2h"], "note": "pinned cudaMemcpyAsync, 256 MiB, this box"},
        "cr": nbytes / blob_len, "blob_bytes": sizes, "max_err_over_eb": max_err / (cfg["eb"] * rng_),
        "gpu_launches": launches,
        "roofline": roofline,
        "kernels": {k: {"launches": v[0] / K, "ms": v[1] / K, "gbs": v[2] / max(v[1], 1e-9) / 1e6} for k, v in
                    sorted(kern.items(), key=lambda kv: -kv[1][1])},
        "decompress_kernels": {k: {"launches": v[0] / K, "ms": v[1] / K, "gbs": v[2] / max(v[1], 1e-9) / 1e6}
                               for k, v in sorted(dkern.items(), key=lambda kv: -kv[1][1])},
        "clocks": clocks,
    }
    if zrate:
        assert bytes(z_host.numpy()) == z_blob, "fixed-rate e2e stream differs from the device-path stream"
        zerr = float(np.max(np.abs(h_out.numpy().astype(np.float64) - a.astype(np.float64))))

        def zroof(kd, name, ms_step):
            nl, kms, kbytes, _ = kd[name]
            ach = (nbytes + z_len) / (kms / nl * 1e-3) / 1e9     # algorithmic: field + stream, once
            return {"bound": "hbm", "kernel": name, "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                    "traffic": ncu_traffic(name), "algorithmic_bytes": nbytes + z_len, "launch_ms": kms / nl,
                    "launches_per_step": nl / K, "share_of_step": kms / (ms_step * K)}

        t_zc = max(nbytes / (pcie["h2d"] * 1e9), z_len / (pcie["d2h"] * 1e9))
        t_zd = max(z_len / (pcie["h2d"] * 1e9), nbytes / (pcie["d2h"] * 1e9))
        line["zfp"] = {
            "mode": f"fixed-rate block coder (hpdr/zfp.py), rate {zrate} bits/value, reference-identical stream",
            "rate": zrate, "stream_bytes": z_len, "cr": nbytes / z_len, "max_abs_err": zerr,
            "compress_gbs": gbs(zc_ms), "compress_ms": zc_ms, "decompress_gbs": gbs(zd_ms), "decompress_ms": zd_ms,
            "gpu_launches_compress": zc_l, "gpu_launches_decompress": zd_l,
            "compress_e2e": {"value": gbs(zce_ms), "unit": "GB/s", "h2d_bytes_per_step": nbytes,
                             "d2h_bytes_per_step": z_len, "ms_per_step": zce_ms,
                             "pcie_roofline_frac": t_zc / (zce_ms * 1e-3)},
            "decompress_e2e": {"value": gbs(zde_ms), "unit": "GB/s", "h2d_bytes_per_step": z_len,
                               "d2h_bytes_per_step": nbytes, "ms_per_step": zde_ms,
                               "pcie_roofline_frac": t_zd / (zde_ms * 1e-3)},
            "pipeline": {"mode": "streams pipeline, ~64 MB chunks, HPDR container (pipeline id 1)",
                         "container_bytes": zp_len, "compress_e2e_gbs": gbs(zpc_ms), "compress_ms": zpc_ms,
                         "decompress_e2e_gbs": gbs(zpd_ms), "decompress_ms": zpd_ms,
                         "compress_pcie_roofline_frac": max(nbytes / (pcie["h2d"] * 1e9),
                                                            zp_len / (pcie["d2h"] * 1e9)) / (zpc_ms * 1e-3),
                         "decompress_pcie_roofline_frac": max(zp_len / (pcie["h2d"] * 1e9),
                                                              nbytes / (pcie["d2h"] * 1e9)) / (zpd_ms * 1e-3)},
            "roofline_encode": zroof(zkern, "k_zfp_encode", zc_ms),
            "roofline_decode": zroof(zdkern, "k_zfp_decode", zd_ms),
        }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if zrate:
            zb = cpu_zfp_time(a, zrate)
            line["zfp"]["cpu_baseline"] = {"value": zb["compress_gbs"], "unit": "GB/s", "cores": zb["cores"],
                                           "kind": "port", "sample": zb["sample"],
                                           "decompress_value": zb["decompress_gbs"]}
        cb = cpu_oracle_time(cfg, a)
        line["cpu_baseline"] = {"value": cb["compress_gbs"], "unit": "GB/s", "cores": cb["cores"], "kind": "port",
                                "sample": cb["sample"], "decompress_value": cb["decompress_gbs"]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
