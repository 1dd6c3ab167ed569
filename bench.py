#!/usr/bin/env python
"""Benchmark of the B200 MGARD reduction path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config target]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

Workload (default ``target``): the north-star Target, one 1024^3 fp32 smooth+noise field, relative
L-inf bound 1e-4, block-partitioned along dim 0 across the N ranks (strong scaling: rank r owns
planes [r*1024/N, (r+1)*1024/N) of the same field and builds only those).  One step = one
``mgard_compress`` of every rank's block, the reference's drop-in call, with the job-wide min/max
all-reduce (16 bytes) inside the call (partition.RangeExchange) at every N, N = 1 included.
Rank 0 prints one JSON line:

  value / e2e  end-to-end compress GB/s: pinned host input -> H2D -> kernels -> D2H of the blob
               into pinned host memory, whole job (input bytes of all ranks / max-over-ranks time)
  decompress   the mirror direction end to end (blob in pinned host memory -> field in pinned host
               memory), plus both directions kernel-only (device-resident in / out)
  roofline     the dominant kernel of the kernel-only compress: algorithmic bytes / CUDA-event
               duration vs the measured HBM peak; traffic from this config's ncu capture
  parity       sha256 of the timed blob and of the decompressed field against reference-pinned
               hashes (tests/golden/), and max error / error bound of the timed decompress output
  cpu_baseline the C port of the reference algorithm (oracle/) on this host's cores (rank 0, N = 1)

Secondary legs (same JSON line): the paper's chunked streams pipeline (M2), the drop-in with pageable
numpy / bytes buffers, the fixed-rate block coder, and configs[1] (513^3) end to end.
"""
from __future__ import annotations

import argparse
import hashlib
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
    "target": dict(workload="north-star Target: 3D fp32 1024^3 smooth+noise field, rel L-inf 1e-4, one field "
                            "block-partitioned along dim 0 across the GPUs (strong scaling)",
                   shape=(1024, 1024, 1024), dtype="f32", field="smooth", eb=1e-4,
                   pin="T_smooth1024_f32_rel1e-4"),
    "c2": dict(workload="configs[1]: 3D fp32 513^3 smooth+noise field, rel L-inf 1e-4", shape=(513, 513, 513),
               dtype="f32", field="smooth", eb=1e-4, pin="C2_smooth513_rel1e-4"),
    "c1": dict(workload="configs[0]: 3D fp32 129^3 GRF, abs L-inf 1e-3", shape=(129, 129, 129), dtype="f32",
               field="grf", eb=1e-3, value_range=(0.0, 1.0), pin="C1_grf129_abs1e-3"),
    "c3": dict(workload="configs[2]: NYX-like 512^3 fp32 temperature, rel 1e-3", shape=(512, 512, 512), dtype="f32",
               field="temperature", eb=1e-3, pin="C3_temperature_512_0.001"),
    "c4": dict(workload="configs[3]: 3D fp64 1024^3 smooth+noise field block-partitioned across the GPUs, "
                        "global range, rel 1e-4 (the L2 request uses the same quantizer, SURVEY 8c)",
               shape=(1024, 1024, 1024), dtype="f64", field="smooth", eb=1e-4, pin="C4_smooth1024_f64"),
    "c5": dict(workload="configs[4]: 1024^3 fp32 timestep, rel 1e-2", shape=(1024, 1024, 1024), dtype="f32",
               field="smooth", eb=1e-2),
}


def block_bounds(n0, world, rank):
    from paper_2503_06322_b200.container import slab_bounds

    return slab_bounds(n0, world, rank)


def make_block(cfg, world, rank):
    """This rank's dim-0 block of the config's field (seed 0: every rank slices the SAME field)."""
    from paper_2503_06322_b200 import synthetic as S

    dt = np.float32 if cfg["dtype"] == "f32" else np.float64
    lo, hi = block_bounds(cfg["shape"][0], world, rank)
    if cfg["field"] == "smooth":
        return S.smooth_noise(cfg["shape"], seed=0, dtype=dt, planes=(lo, hi) if world > 1 else None)
    if cfg["field"] == "grf":
        a = S.grf(cfg["shape"], m=8, seed=0, dtype=dt)
    else:
        a = S.nyx_like(cfg["shape"], cfg["field"], seed=None, dtype=dt)
    return np.ascontiguousarray(a[lo:hi]) if world > 1 else a


def load_pins():
    pins = {}
    for f in ("configs.json", "scale_pins.json"):
        p = os.path.join(ROOT, "tests", "golden", f)
        if os.path.exists(p):
            with open(p) as fh:
                pins.update(json.load(fh))
    return pins


def pin_for(cfg, world, rank, pins):
    """The reference-pinned hashes of this rank's block, if any."""
    name = cfg.get("pin")
    if not name:
        return None
    if cfg["field"] == "smooth" and cfg["dtype"] == "f64":   # C4: slabs k of N
        return pins.get(f"{name}_slab{rank}of{world}")
    return pins.get(name) if world == 1 else None


def config_dict(cfg, world):
    """The config keys both arms print (identical, so the driver can pair the lines)."""
    return {"workload": cfg["workload"], "shape": list(cfg["shape"]), "input_dtype": cfg["dtype"],
            "eb_rel": cfg["eb"], "value_range": list(cfg["value_range"]) if cfg.get("value_range") else None,
            "partition": f"dim-0 blocks x{world}, job-wide range", "direction": "compress (decompress beside)"}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(config, kernel):
    """DRAM bytes (read + write) of one launch of `kernel` from this config's committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        return t.get(config, {}).get(kernel)
    except Exception:
        return None


def pcie_roofline(dev, mib=256):
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
            for _ in range(3):
                fn()
            e1.record()
            e1.synchronize()
            best = max(best, n * 3 / (e0.elapsed_time(e1) * 1e-3) / 1e9)
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


# ----------------------------------------------------------------------------- CPU arms
def cpu_oracle_time(cfg, a, budget_s=20.0, value_range=None):
    """Time the C port of the reference algorithm on this host's cores, on a bounded slab sample."""
    from oracle import oracle as O

    threads = os.cpu_count() or 1
    O.set_threads(threads)
    vr = value_range or cfg.get("value_range")
    planes = min(a.shape[0], 17)
    t0 = time.perf_counter()
    O.mgard_compress(np.ascontiguousarray(a[:planes]), cfg["eb"], value_range=vr)
    per_plane = (time.perf_counter() - t0) / planes
    planes = int(max(9, min(a.shape[0], budget_s / 3.0 / max(per_plane, 1e-9))))
    sample = np.ascontiguousarray(a[:planes])
    reps, tc, td = 0, 0.0, 0.0
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
                sample=f"first {planes} of {a.shape[0]} planes of the workload ({sample.nbytes / 1e6:.0f} MB) x {reps}, "
                       f"C oracle (port of hpdr/mgard), OpenMP {threads} threads")


def reference_python_time(cfg, a, planes=8):
    """The reference itself (baseline/_ref: hpdr.mgard, numpy + numba, SerialAdapter), 1 core, on the
    first `planes` planes of the workload."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "hpdr")):
        return {"unavailable": "baseline/_ref not installed"}
    env = dict(os.environ, PYTHONPATH=ref, NUMBA_CACHE_DIR=os.path.join(tempfile.gettempdir(), "hpdr_numba"),
               OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1", NUMBA_NUM_THREADS="1")
    sample = np.ascontiguousarray(a[:min(planes, a.shape[0])])
    with tempfile.NamedTemporaryFile(suffix=".npy", delete=False) as f:
        np.save(f, sample)
        path = f.name
    vr = cfg.get("value_range")
    code = f"""
import json, os, time, numpy as np
os.sched_setaffinity(0, {{min(os.sched_getaffinity(0))}})
from hpdr.exec_core.tensor import TensorData, DType
from hpdr.mgard import mgard_compress, mgard_decompress
a = np.load({path!r})
td = lambda x: TensorData(tuple(x.shape), DType.F32 if x.dtype == np.float32 else DType.F64, x)
w = np.ascontiguousarray(a[:1, :33, :33])
mgard_decompress(mgard_compress(td(w), {cfg['eb']!r}, value_range={vr!r}))   # numba JIT warm-up
t0 = time.perf_counter(); b = mgard_compress(td(a), {cfg['eb']!r}, value_range={vr!r}); t1 = time.perf_counter()
mgard_decompress(b); t2 = time.perf_counter()
print(json.dumps({{"c": t1 - t0, "d": t2 - t1, "n": a.nbytes}}))
"""
    try:
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        res = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:   # noqa: BLE001
        return {"unavailable": f"reference run failed: {type(e).__name__}"}
    finally:
        os.unlink(path)
    return {"compress_gbs": res["n"] / res["c"] / 1e9, "decompress_gbs": res["n"] / res["d"] / 1e9, "cores": 1,
            "kind": "reference",
            "sample": f"first {sample.shape[0]} planes ({res['n'] / 1e6:.1f} MB), hpdr.mgard from baseline/_ref "
                      f"(numpy + numba, SerialAdapter), one core, warm JIT"}


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    a = make_block(cfg, 1, 0)
    from oracle import oracle as O

    threads = os.cpu_count() or 1
    O.set_threads(threads)
    vr = cfg.get("value_range")
    planes = min(a.shape[0], 17)
    t0 = time.perf_counter()
    O.mgard_compress(np.ascontiguousarray(a[:planes]), cfg["eb"], value_range=vr)
    per_plane = (time.perf_counter() - t0) / planes
    # bound the whole --steps K --warmup W run to ~2 minutes of CPU work
    budget_step = 100.0 / max(1, args.steps + args.warmup)
    planes = int(max(9, min(a.shape[0], budget_step / max(per_plane, 1e-9))))
    sample = np.ascontiguousarray(a[:planes])
    for _ in range(args.warmup):
        O.mgard_compress(sample, cfg["eb"], value_range=vr)
    t0 = time.perf_counter()
    blob = None
    for _ in range(args.steps):
        blob = O.mgard_compress(sample, cfg["eb"], value_range=vr)
    dt = time.perf_counter() - t0
    t1 = time.perf_counter()
    O.mgard_decompress(blob)
    ddt = time.perf_counter() - t1
    v = sample.nbytes * args.steps / dt / 1e9
    py = reference_python_time(cfg, a)
    line = {"metric": METRIC, "impl": "reference", "value": v, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, SIMD-invariant generators)", "config": config_dict(cfg, world),
            "decompress": {"value": sample.nbytes / ddt / 1e9, "unit": "GB/s"},
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": threads, "kind": "port",
                             "sample": f"first {planes} of {a.shape[0]} planes per step, C oracle port of "
                                       f"hpdr/mgard (OpenMP {threads} threads), rank 0 only",
                             "decompress_value": sample.nbytes / ddt / 1e9},
            "reference_python_1core": py,
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="target", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the M2 / pageable / fixed-rate / 513^3 legs")
    ap.add_argument("--zfp-rate", type=int, default=16, help="bits/value of the fixed-rate leg (0: skip)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    same_gpu = os.environ.get("HPDR_BENCH_SAME_GPU") == "1"   # multi-rank path on a 1-GPU box
    if same_gpu:
        local = 0
    from paper_2503_06322_b200 import numa

    numa_info = numa.bind_to_gpu(local) if world > 1 and not same_gpu else {"node": None}

    import torch
    import torch.distributed as dist

    import paper_2503_06322_b200 as P
    from paper_2503_06322_b200 import _lib
    from paper_2503_06322_b200 import pipeline as PL
    from paper_2503_06322_b200 import synthetic as S
    from paper_2503_06322_b200.partition import RangeExchange, allreduce_range

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if not same_gpu else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if not same_gpu else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    pins = load_pins()
    a = make_block(cfg, world, rank)                     # this rank's block of the one field
    pin = pin_for(cfg, world, rank, pins)
    input_ok = pin is None or S.sha256(a) == pin["input_sha"]
    nbytes = a.nbytes
    total_in = sum_over_ranks(nbytes)
    ctx = _lib.default_context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    tdt = torch.float32 if a.dtype == np.float32 else torch.float64
    h_in = torch.from_numpy(a).pin_memory()               # pinned host input (e2e legs)
    d_in = h_in.to(dev)                                   # HBM-resident input (kernel-only legs)
    vr_cfg = cfg.get("value_range")
    rx = RangeExchange(ctx, group=None if not same_gpu else None)

    def compress(src, out):
        """The timed call: relative mode with the job-wide range exchanged inside it (or the
        config's absolute range)."""
        if vr_cfg is not None:
            return P.mgard_compress(src, cfg["eb"], value_range=vr_cfg, out=out)
        with rx:
            return P.mgard_compress(src, cfg["eb"], out=out)

    # ---- M1 outputs: every leg owns its buffers
    cap = int(nbytes * 1.3) + (16 << 20)
    d_blob_out = torch.empty(cap, dtype=torch.uint8, device=dev)
    blob_len = compress(d_in, d_blob_out)
    vr_job = vr_cfg or rx.last                            # the range the blobs were made with
    blob_dev = bytes(d_blob_out[:blob_len].cpu().numpy())
    h_blob = torch.empty(cap, dtype=torch.uint8).pin_memory()
    h_blob_in = torch.from_numpy(np.frombuffer(blob_dev, np.uint8).copy()).pin_memory()
    d_blob_in = h_blob_in.to(dev)
    h_out = torch.empty(a.shape, dtype=tdt).pin_memory()
    d_out = torch.empty(a.shape, dtype=tdt, device=dev)

    def compress_e2e():
        return compress(h_in, h_blob)

    def compress_dev():
        return compress(d_in, d_blob_out)

    def decompress_e2e():
        P.mgard_decompress(h_blob_in, out=h_out)

    def decompress_dev():
        P.mgard_decompress(d_blob_in, out=d_out)

    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev) if nbytes < (126 << 20) else None

    def timed(fn, steps, prof=False):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize(dev)
        barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        _lib.launch_count(reset=True)
        if prof:
            _lib.prof_enable(prof)
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
        return max_over_ranks(total) / steps, launches, kern

    K = args.steps
    pcie = pcie_roofline(dev)
    sec = {}
    with ClockSampler(local) as clk:
        e_ms, e_launch, _ = timed(compress_e2e, K)
        de_ms, de_launch, _ = timed(decompress_e2e, K)
        c_ms, c_launch, kern = timed(compress_dev, K, prof=True)
        d_ms, _, _ = timed(decompress_dev, K)
        # per-kernel decompress times from a serialized pass (side-stream kernels would overlap)
        _, _, dkern = timed(decompress_dev, 1, prof="serial")
        if not args.no_secondary:
            sec = secondary_legs(args, cfg, a, h_in, d_in, vr_job, timed, world, rank, pins, dev)
    clocks = clk.summary()

    # ---- parity of what was timed (every rank checks its own block)
    blob_e2e = bytes(h_blob[:blob_len].numpy())
    out_e2e = h_out.numpy()
    rng_ = vr_job[1] - vr_job[0]
    max_err = float(np.max(np.abs(out_e2e.astype(np.float64) - a.astype(np.float64))))
    err_over_eb = max_err / (cfg["eb"] * rng_) if rng_ > 0 else 0.0
    checks = {"input_sha_matches_pin": input_ok if pin else None,
              "e2e_blob_equals_device_blob": blob_e2e == blob_dev,
              "blob_sha_matches_pin": (hashlib.sha256(blob_e2e).hexdigest() == pin["blob_sha"]) if pin else None,
              "out_sha_matches_pin": (S.sha256(out_e2e) == pin["out_sha"]) if pin else None,
              "device_out_equals_e2e_out": bool(np.array_equal(d_out.cpu().numpy().view(np.uint8),
                                                               out_e2e.view(np.uint8))),
              "max_err_over_eb": err_over_eb}
    ok = (checks["e2e_blob_equals_device_blob"] and checks["device_out_equals_e2e_out"] and err_over_eb <= 1.0
          and all(v is not False for k, v in checks.items() if k.endswith("pin")))
    all_ok = max_over_ranks(0.0 if ok else 1.0) == 0.0
    worst_err = max_over_ranks(err_over_eb)
    sizes = [blob_len]
    if world > 1:
        g = [None] * world
        dist.all_gather_object(g, {"blob": blob_len, "checks": checks, "pin": pin["name"] if pin else None})
        sizes = [x["blob"] for x in g]
        rank_checks = g
    else:
        rank_checks = [{"blob": blob_len, "checks": checks, "pin": pin["name"] if pin else None}]
    total_blob = sum(sizes)
    gbs = lambda ms: total_in / (ms * 1e-3) / 1e9  # noqa: E731

    hbm, peak_kind = measured_peaks()
    dname, (dl, dms, dbytes, dmax) = max(kern.items(), key=lambda kv: kv[1][1])
    achieved = dbytes / (dms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": ncu_traffic(args.config, dname),
                "algorithmic_bytes": dbytes / max(dl, 1), "launch_ms": dms / max(dl, 1), "peak_kind": peak_kind,
                "share_of_step": dms / (c_ms * K), "launches_per_step": dl / K,
                "timing": "CUDA events on the launching stream around every launch of the kernel in the timed "
                          "kernel-only compress steps (rank 0)",
                "traffic_source": f"profiles/ncu_traffic.json[{args.config!r}] (ncu --set full, "
                                  "dram__bytes_read+write per launch); null when not captured for this config"}
    # probed again after the timed legs, the better of the two per direction (one box's first probe
    # read 48 GB/s H2D while its M1 compress streamed at 55)
    pcie2 = pcie_roofline(dev)
    pcie = {k: max(pcie[k], pcie2[k]) for k in pcie}
    # end-to-end roofline: the copies alone at the measured pinned PCIe rates (per rank: its own bytes)
    t_c = max(nbytes / (pcie["h2d"] * 1e9), blob_len / (pcie["d2h"] * 1e9))
    t_d = max(blob_len / (pcie["h2d"] * 1e9), nbytes / (pcie["d2h"] * 1e9))
    t_c, t_d = max_over_ranks(t_c), max_over_ranks(t_d)

    line = {
        "metric": METRIC, "value": gbs(e_ms), "unit": "GB/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": e_ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SIMD-invariant generators)",
        "config": config_dict(cfg, world),
        "timing": "CUDA events around each step on the context's stream, max over ranks; "
                  + ("inputs larger than L2 (no flush needed)" if flush is None
                     else "inputs smaller than L2: 256 MB buffer written between separately timed steps"),
        "e2e": {"value": gbs(e_ms), "unit": "GB/s", "h2d_bytes_per_step": int(total_in),
                "d2h_bytes_per_step": int(total_blob), "ms_per_step": e_ms,
                "memory": "pinned host in / out, mgard_compress(tensor, eb_rel, out=pinned) per rank",
                "pcie_roofline_frac": t_c / (e_ms * 1e-3), "gpu_launches_per_step": e_launch / K},
        "decompress": {"e2e": {"value": gbs(de_ms), "unit": "GB/s", "h2d_bytes_per_step": int(total_blob),
                               "d2h_bytes_per_step": int(total_in), "ms_per_step": de_ms,
                               "pcie_roofline_frac": t_d / (de_ms * 1e-3)},
                       "kernel_only": {"value": gbs(d_ms), "ms_per_step": d_ms}},
        "kernel_only": {"value": gbs(c_ms), "ms_per_step": c_ms,
                        "note": "device-resident input, blob left in device memory"},
        "pcie": {"h2d_gbs": pcie["h2d"], "d2h_gbs": pcie["d2h"], "note": "pinned cudaMemcpyAsync, 256 MiB, this box, best of a probe before and after the timed legs"},
        "cr": total_in / total_blob, "blob_bytes": sizes, "value_range": list(vr_job),
        "parity": {"ok": all_ok, "max_err_over_eb": worst_err, "ranks": rank_checks},
        "gpu_launches": e_launch,
        "roofline": roofline,
        "kernels": {k: {"launches": v[0] / K, "ms": v[1] / K, "gbs": v[2] / max(v[1], 1e-9) / 1e6} for k, v in
                    sorted(kern.items(), key=lambda kv: -kv[1][1])},
        "decompress_kernels": {
            "note": "per-kernel CUDA events from one separate decompress with the device synchronized around "
                    "every launch (hpdr_prof_enable(2)): no overlap, so they add up; the step time is unprofiled",
            **{k: {"launches": v[0], "ms": v[1], "gbs": v[2] / max(v[1], 1e-9) / 1e6}
               for k, v in sorted(dkern.items(), key=lambda kv: -kv[1][1])}},
        "clocks": clocks,
        "numa": numa_info,
        **sec,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_oracle_time(cfg, a, value_range=vr_cfg)
        line["cpu_baseline"] = {"value": cb["compress_gbs"], "unit": "GB/s", "cores": cb["cores"], "kind": "port",
                                "sample": cb["sample"], "decompress_value": cb["decompress_gbs"]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    if not all_ok:
        sys.exit(3)


def secondary_legs(args, cfg, a, h_in, d_in, vr_job, timed, world, rank, pins, dev):
    """M2 pipeline, pageable drop-in, fixed-rate coder and (default config) the 513^3 config, end to end."""
    import torch

    import paper_2503_06322_b200 as P
    from paper_2503_06322_b200 import pipeline as PL
    from paper_2503_06322_b200 import synthetic as S
    from paper_2503_06322_b200 import zfp as ZF

    K = args.steps
    nbytes = a.nbytes
    out = {}

    def gbs_job(ms):
        return nbytes * world / (ms * 1e-3) / 1e9

    # M2: the paper's chunked streams pipeline (HPDR container of per-chunk reference blobs), with
    # the job-wide range given (each chunk = mgard_compress(chunk, eb, value_range=job range))
    pipe_out = torch.empty(int(nbytes * 1.3) + (64 << 20), dtype=torch.uint8).pin_memory().numpy()
    chunk_planes = max(1, (64 << 20) // a[0].nbytes)
    pipe_len = PL.compress_pipelined(h_in, cfg["eb"], value_range=vr_job, chunk_planes=chunk_planes, out=pipe_out)
    pipe_in = torch.from_numpy(pipe_out[:pipe_len].copy()).pin_memory().numpy()
    pipe_dec = torch.empty(a.shape, dtype=h_in.dtype).pin_memory().numpy()
    pc_ms, _, _ = timed(lambda: PL.compress_pipelined(h_in, cfg["eb"], value_range=vr_job, chunk_planes=chunk_planes,
                                                      out=pipe_out), K)
    pd_ms, _, _ = timed(lambda: PL.decompress_pipelined(pipe_in, out=pipe_dec), K)
    m2 = {"mode": f"M2 streams pipeline, {chunk_planes}-plane chunks, 3 queues, job-wide value_range",
          "compress_e2e_gbs": gbs_job(pc_ms), "decompress_e2e_gbs": gbs_job(pd_ms), "compress_ms": pc_ms,
          "decompress_ms": pd_ms, "cr": nbytes / pipe_len}
    from paper_2503_06322_b200.container import read_container

    h, payloads = read_container(pipe_out[:pipe_len])
    pin = pins.get(cfg.get("pin")) if world == 1 else None
    if pin and pin.get("m2_chunk_sha") and pin.get("m2_chunk_planes") == chunk_planes:
        m2["chunks_match_pin"] = [hashlib.sha256(bytes(p)).hexdigest() for p in payloads] == pin["m2_chunk_sha"]
    m2["decompressed_equals_input_bound"] = float(np.max(np.abs(pipe_dec.astype(np.float64) - a))) <= \
        cfg["eb"] * (vr_job[1] - vr_job[0])
    out["pipeline"] = m2

    # the drop-in exactly as a reference user calls it: numpy array in, Python bytes out (and back).
    # Steady state: the reused input array is page-locked on its second use and decompressed arrays
    # come from the pinned pool (hostmem.py); "no_hostmem": the same calls with both caches off
    # (every call staged through the pinned rings, fresh result array) -- a one-shot call's cost.
    from paper_2503_06322_b200 import hostmem

    blob_np = P.mgard_compress(a, cfg["eb"], value_range=vr_job)
    pg_c_ms, _, _ = timed(lambda: P.mgard_compress(a, cfg["eb"], value_range=vr_job), K)
    pg_d_ms, _, _ = timed(lambda: P.mgard_decompress(blob_np), K)
    hostmem.enabled = False
    try:
        ng_c_ms, _, _ = timed(lambda: P.mgard_compress(a, cfg["eb"], value_range=vr_job), K)
        ng_d_ms, _, _ = timed(lambda: P.mgard_decompress(blob_np), K)
    finally:
        hostmem.enabled = True
    out["pageable"] = {"mode": "drop-in API with a numpy array in / Python bytes out (pageable host memory), "
                               "steady state: reused input page-locked, result arrays from the pinned pool",
                       "compress_e2e_gbs": gbs_job(pg_c_ms), "decompress_e2e_gbs": gbs_job(pg_d_ms),
                       "compress_ms": pg_c_ms, "decompress_ms": pg_d_ms,
                       "blob_equals_pinned_path": blob_np == bytes(P.mgard_compress(h_in, cfg["eb"], value_range=vr_job)),
                       "no_hostmem": {"compress_e2e_gbs": gbs_job(ng_c_ms), "decompress_e2e_gbs": gbs_job(ng_d_ms),
                                      "compress_ms": ng_c_ms, "decompress_ms": ng_d_ms},
                       "hostmem_alloc_events": hostmem.alloc_events()}

    # fixed-rate block coder (hpdr/zfp.py) on the same block, its own buffers
    zrate = args.zfp_rate if a.ndim <= 3 else 0
    if zrate:
        code = 0 if a.dtype == np.float32 else 1
        z_len = ZF.compressed_size(a.shape, P.DType.F32 if code == 0 else P.DType.F64, zrate)
        z_dev = torch.empty(z_len, dtype=torch.uint8, device=dev)
        z_host = torch.empty(z_len, dtype=torch.uint8).pin_memory()
        z_out_d = torch.empty(a.shape, dtype=h_in.dtype, device=dev)
        z_out_h = torch.empty(a.shape, dtype=h_in.dtype).pin_memory()
        ZF.zfp_compress(d_in, zrate, out=z_dev)
        z_blob = bytes(z_dev.cpu().numpy())
        z_host_in = torch.from_numpy(np.frombuffer(z_blob, np.uint8).copy()).pin_memory()
        zc_ms, _, _ = timed(lambda: ZF.zfp_compress(d_in, zrate, out=z_dev), K)
        zd_ms, _, _ = timed(lambda: ZF.zfp_decompress(z_dev, out=z_out_d), K)
        zce_ms, _, _ = timed(lambda: ZF.zfp_compress(h_in, zrate, out=z_host), K)
        zde_ms, _, _ = timed(lambda: ZF.zfp_decompress(z_host_in, out=z_out_h), K)
        out["zfp"] = {"mode": f"fixed-rate block coder (hpdr/zfp.py), rate {zrate} bits/value",
                      "stream_bytes": z_len, "cr": nbytes / z_len,
                      "compress_gbs": gbs_job(zc_ms), "decompress_gbs": gbs_job(zd_ms),
                      "compress_e2e_gbs": gbs_job(zce_ms), "decompress_e2e_gbs": gbs_job(zde_ms),
                      "e2e_stream_equals_device_stream": bytes(z_host.numpy()) == z_blob,
                      "e2e_out_equals_device_out": bool(np.array_equal(z_out_h.numpy().view(np.uint8),
                                                                       z_out_d.cpu().numpy().view(np.uint8))),
                      "max_abs_err": float(np.max(np.abs(z_out_h.numpy().astype(np.float64) - a)))}

    # configs[1] (513^3 fp32, rel 1e-4) end to end beside the Target, pinned to the reference's hashes
    if args.config == "target" and world == 1:
        c2 = CONFIGS["c2"]
        b = make_block(c2, 1, 0)
        pb = pins.get(c2["pin"])
        hb = torch.from_numpy(b).pin_memory()
        hblob = torch.empty(int(b.nbytes * 1.3) + (16 << 20), dtype=torch.uint8).pin_memory()
        hout = torch.empty(b.shape, dtype=torch.float32).pin_memory()
        n = P.mgard_compress(hb, c2["eb"], out=hblob)
        blob = bytes(hblob[:n].numpy())
        hbin = torch.from_numpy(np.frombuffer(blob, np.uint8).copy()).pin_memory()
        c_ms, _, _ = timed(lambda: P.mgard_compress(hb, c2["eb"], out=hblob), K)
        d_ms, _, _ = timed(lambda: P.mgard_decompress(hbin, out=hout), K)
        out["configs_1_513"] = {
            "workload": c2["workload"], "compress_e2e_gbs": b.nbytes / (c_ms * 1e-3) / 1e9,
            "decompress_e2e_gbs": b.nbytes / (d_ms * 1e-3) / 1e9, "compress_ms": c_ms, "decompress_ms": d_ms,
            "cr": b.nbytes / n,
            "blob_sha_matches_reference": hashlib.sha256(bytes(hblob[:n].numpy())).hexdigest() == pb["blob_sha"]
            if pb else None,
            "out_sha_matches_reference": S.sha256(hout.numpy()) == pb["out_sha"] if pb else None}
    return out


if __name__ == "__main__":
    main()
