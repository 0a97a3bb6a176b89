"""Benchmark: FST eval points/s (fp64) + randomized-LS core refit seconds.

Workload (BASELINE.json configs[1] = "C2"): 16,777,216 points on a jittered
256^3 mesh (seeded), flame-front field + 8 Gaussians + N(0, 1e-4) noise; a
functional sparse Tucker model with ranks (32,32,32), Legendre degree 48,
<= 24 nonzeros per function, fitted from seed by the upstream stand-in
(synth.fitted_model); refit with M = 8R = 262,144 sketch rows (DCT).

A step = one evaluation of all N points of this rank (weak scaling: every
rank evaluates its own N points).  `value` is device-timed with the points
already in HBM (inputs 384 MB > 126 MB L2, so no flush is needed); `e2e` is
the same metric through the host C-ABI call (pinned host buffers, H2D of the
points and D2H of the values inside the timed region).  The refit (one
problem, rows sharded across ranks + one NCCL all-reduce of A^T A) reports
the median of --refit-reps (default 3) timed refits after --refit-warmup
(default 1) untimed full-size refits, like the W warm-up steps of the
evaluation; the first (cold) run is reported beside it under "refit"."cold",
and one further refit with per-kernel event profiling gives the stage
breakdown.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FST eval points/s (fp64) + randomized-LS core refit s, at 1/2/4/8 B200"
UNIT = "points/s"


DATA_DESC = {
    "C1": "synthetic (seeded uniform points in [0,1]^3, analytic flame field; model fitted from "
          "seed by the upstream stand-in on a 64^3 grid)",
    "C2": "synthetic (seeded jittered 256^3 mesh, analytic flame field; model fitted from seed by "
          "the upstream stand-in)",
    "C3": "synthetic (seeded points, 50% uniform and 50% within 0.03 of the flame surface; seeded "
          "random model of the config's shape)",
    "C4": "synthetic (seeded 4D points, t on 64 snapshots, travelling-front field; seeded random "
          "model of the config's shape)",
    "C5": "synthetic (seeded uniform points shared by 8 seeded random models of the config's "
          "shape)",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--points", type=int, default=0, help="override N per rank")
    ap.add_argument("--no-refit", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--transform", default="dct")
    ap.add_argument("--no-refit-none", action="store_true",
                    help="skip the transform='none' refit reported as refit_none")
    ap.add_argument("--refit-reps", type=int, default=3,
                    help="timed refits; the line reports their median")
    ap.add_argument("--refit-warmup", type=int, default=1,
                    help="untimed full-size refits before the timed one (cuBLASLt algorithm "
                         "choice per Gram shape, lazy kernel loading)")
    return ap.parse_args()


# ------------------------------------------------------------- workload ---
def dataset(cfg_name: str, n_override: int, rank: int):
    """Seeded points (Q x d, column-major) and values (or None) of a config;
    `rank` offsets the seed (each rank's own weak-scaling slab)."""
    from paper_1907_05884_b200 import synth

    c = synth.CONFIGS[cfg_name]
    seed = 0
    if cfg_name == "C2":
        n = n_override or 256 ** 3
        pts = synth.jittered_mesh(256, seed=seed + 1000 * rank) if not n_override else \
            synth.uniform_points(n, 3, seed + 1000 * rank)
        vals = synth.flame_field(pts, seed=seed, n_gauss=8, noise=1e-2)
    elif cfg_name == "C1":
        n = n_override or c["n"]
        pts = synth.uniform_points(n, 3, seed + 1000 * rank)
        vals = synth.flame_field(pts, seed=seed, noise=1e-2)
    elif cfg_name == "C4":
        # 4D space-time: x, y, z uniform, t on 64 uniform snapshots; the
        # travelling front of BASELINE configs[3]; refit with M = 16R.
        n = n_override or min(c["n"], 1 << 24)
        rng = np.random.default_rng(seed + 1000 * rank)
        pts = rng.random((n, 4))
        pts[:, 3] = rng.integers(0, 64, n) / 63.0
        x, y, z, t = pts[:, 0], pts[:, 1], pts[:, 2], pts[:, 3]
        vals = np.tanh((z - 0.3 - 0.4 * t - 0.05 * np.sin(2 * np.pi * x) * np.sin(2 * np.pi * y))
                       / 0.02)
    else:
        n = n_override or min(c["n"], 1 << 24)
        d = c["d"]
        pts = synth.uniform_points(n, d, seed + 1000 * rank) if d == 4 or cfg_name == "C5" else \
            synth.flame_surface_mixture(n, seed + 1000 * rank)
        vals = None
    return np.asfortranarray(pts), vals


def workload(cfg_name: str, n_override: int, rank: int):
    from paper_1907_05884_b200 import synth

    c = synth.CONFIGS[cfg_name]
    seed = 0
    if cfg_name == "C2":
        model = synth.fitted_model(256, c["ranks"], c["degrees"][0], c["nnz"], seed=seed,
                                   n_gauss=8)
    elif cfg_name == "C1":
        model = synth.fitted_model(c["grid"], c["ranks"], c["degrees"][0], c["nnz"], seed=seed)
    else:
        model = synth.random_model(c["ranks"], c["degrees"], c["nnz"], seed=seed)
    pts, vals = dataset(cfg_name, n_override, rank)
    return model, pts, vals, c


def flops_per_point(model) -> tuple[float, float]:
    """F_contract = 2 sum_k prod_{m<k} r_m, F_modes = sum_k (2 nnz_k + 6 p_k)."""
    r = model.ranks
    fc = 2.0 * sum(float(np.prod(r[:k + 1])) for k in range(len(r)))
    fm = 0.0
    for k, mode in enumerate(model.modes):
        nnz = sum(len(fn.coeffs) for fn in mode)
        p = max(fn.basis.degree for fn in mode)
        fm += 2.0 * nnz + 6.0 * p
    return fc, fm


# ------------------------------------------------------------------ clocks ---
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.proc = None
        self.path = os.path.join("/tmp", f"fstk_clocks_{os.getpid()}.csv")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict | None:
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 7:
                    continue
                try:
                    sm.append(float(f[0]))
                    mx = max(mx, float(f[1]))
                except ValueError:
                    continue
                for nm, v in zip(names, f[3:7]):
                    if v.lower() == "active":
                        reasons.add(nm)
            os.unlink(self.path)
        except Exception:
            pass
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------- helpers ---
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def maxreduce(x: float, world: int, device) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_eval_baseline(model, pts, budget_s: float = 12.0) -> dict:
    """Oracle restatement (oracle/liboracle.so) on all host threads, bounded sample."""
    from oracle import oracle as O

    cores = O.max_threads()
    n0 = min(pts.shape[0], 1 << 13)
    t0 = time.perf_counter()
    O.evaluate_batch(model, pts[:n0])
    dt = max(time.perf_counter() - t0, 1e-6)
    n = int(min(pts.shape[0], max(n0, n0 * budget_s / dt)))
    t0 = time.perf_counter()
    O.evaluate_batch(model, pts[:n])
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"first {n} points of this rank's workload, oracle evaluate_batch "
                      f"(restated model.cpp:208-227, parallel_for over {cores} threads), {dt:.1f} s"}


def cpu_refit_estimate(model, pts, vals, S: int, transform: str = "dct") -> dict:
    """Reference refit on the host, EXTRAPOLATED (A alone is 68.7 GB
    at C2 and the QR 5.4e14 flop, infeasible on the host): prepare timed in
    full; the sketch (design column + the reference's DCT, pinned bit-exact to
    its own transforms.cpp, + sampling; parallel over columns like
    solve_sketched) timed on k columns and scaled by (R+1)/k; the QR flop count
    2 m R^2 - 2/3 R^3 at the host's measured pivoted-QR rate (scipy dgeqp3 on
    all threads -- conservative: the reference's Eigen QR is single-threaded)."""
    import scipy.linalg as sla

    from oracle import oracle as O

    cores = O.max_threads()
    R = int(np.prod(model.ranks))
    t0 = time.perf_counter()
    O.refit_columns(model, pts, vals, 0, 0, seed=0, sample_rows=S, transform=transform)
    t_prep = time.perf_counter() - t0
    k = max(2 * cores, 16)
    t0 = time.perf_counter()
    O.refit_columns(model, pts, vals, 0, k, seed=0, sample_rows=S, transform=transform)
    t_k = max(time.perf_counter() - t0 - t_prep, 1e-6)
    t_sketch = t_k / k * (R + 1)
    m_, n_ = 4096, 1024
    a = np.random.default_rng(0).standard_normal((m_, n_))
    sla.qr(a[:512, :128], mode="economic", pivoting=True)
    t0 = time.perf_counter()
    sla.qr(a, mode="economic", pivoting=True)
    rate = (2.0 * m_ * n_ ** 2 - 2.0 / 3.0 * n_ ** 3) / (time.perf_counter() - t0)
    m_rows = 2 * S if transform == "fft" else S
    t_qr = (2.0 * m_rows * R ** 2 - 2.0 / 3.0 * R ** 3) / rate
    return {"seconds": t_prep + t_sketch + t_qr, "extrapolated": True, "kind": "port",
            "cores": cores, "prepare_s": t_prep, "sketch_s": t_sketch, "qr_s": t_qr,
            "qr_gflops_measured": rate / 1e9,
            "sample": f"prepare in full; sketch of {k} of {R + 1} columns scaled; QR "
                      f"{m_rows}x{R} by flop count at the measured {rate / 1e9:.0f} GFLOP/s "
                      f"(dgeqp3 4096x1024, {cores} threads)"}


def traffic_from_profile(cfg: str):
    """dram bytes per contraction launch from the committed ncu capture, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_contract_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        if d.get("config") == cfg:
            return d.get("dram_bytes_per_launch"), d.get("points_per_launch")
    except Exception:
        pass
    return None, None


L2_BYTES = 126 << 20


def arm_config(args, model, cfgd, n: int, nf: int, world: int) -> dict:
    """The `config` of both arms (ours and --impl reference): the workload one
    step processes on each rank, whatever sample the host arm times."""
    in_bytes = n * model.order * 8 + n * 8
    return {"workload": f"{args.config}: evaluate {n} points per rank"
                        + (f" x {nf} fields (value counts field-points)" if nf > 1 else "")
                        + f", ranks {tuple(model.ranks)}, Legendre p={cfgd['degrees'][0]}, "
                          f"<= {cfgd['nnz']} nnz",
            "points_per_rank": n,
            "l2": ("inputs (%d MB) exceed 2x the 126 MB L2; no flush needed" % (in_bytes >> 20))
                  if in_bytes > 2 * L2_BYTES else
                  "L2 flushed between steps (512 MB buffer write, untimed)",
            "parallelism": f"point-sharded x{world}"}


def int8_peak(dev) -> dict:
    """Live int8 x int8 -> int32 GEMM ceiling of this GPU (cuBLASLt through
    torch._int_mm, TN 8192 x 8192 x 16384, best of 5 after warm-up): the
    denominator of the sliced Gram's roofline."""
    import torch

    a = torch.randint(-127, 128, (8192, 16384), dtype=torch.int8, device=dev)
    b = torch.randint(-127, 128, (8192, 16384), dtype=torch.int8, device=dev).t()
    for _ in range(3):
        torch._int_mm(a, b)
    best = float("inf")
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch._int_mm(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    return {"tops": 2.0 * 8192 * 8192 * 16384 / (best * 1e-3) / 1e12,
            "source": "live cuBLASLt int8 TN GEMM 8192x8192x16384 via torch._int_mm, best of 5 "
                      "(burst; MEASURED_PEAKS.json has no int8 entry)"}


# ------------------------------------------------------------ reference arm ---
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O

    model, pts, vals, c = workload(args.config, args.points, 0)
    cores = O.max_threads()
    # each step: a bounded sample (~3 s of CPU work) of the same workload
    n0 = min(pts.shape[0], 1 << 13)
    t0 = time.perf_counter()
    O.evaluate_batch(model, pts[:n0])
    per = (time.perf_counter() - t0) / n0
    n = int(min(pts.shape[0], max(n0, 3.0 / per)))
    for _ in range(args.warmup):
        O.evaluate_batch(model, pts[:min(n, 1 << 12)])
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.evaluate_batch(model, pts[:n])
        times.append(time.perf_counter() - t0)
    ms = 1e3 * float(np.mean(times))
    value = n / (ms * 1e-3)
    nfull = pts.shape[0]
    nf = 8 if args.config == "C5" else 1
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": DATA_DESC.get(args.config, "synthetic"), "impl": "reference",
            "config": arm_config(args, model, c, nfull, nf, world),
            "sample": {"points_per_step": n, "points_in_config": nfull,
                       "full_step_seconds_extrapolated": nfull * nf / value,
                       "note": "each step times the first %d of the %d points of this config "
                               "(per-point cost does not depend on position); a full step "
                               "would take %.1f s on these cores" % (n, nfull, nfull * nf / value)},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{n} of {nfull} points per step of the {args.config} "
                                       "workload; oracle restatement of evaluate_batch (the "
                                       "reference cannot build: Eigen absent), all host threads"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    if vals is not None and not args.no_refit:
        line["refit"] = cpu_refit_estimate(model, pts, vals, c["m_factor"] * int(np.prod(model.ranks)),
                                           args.transform)
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm ---
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    rank, world, local = dist_env()
    import torch

    # One process per GPU; FSTK_BENCH_BACKEND=gloo (with more ranks than GPUs)
    # exercises the multi-rank code path on a single GPU (host-mediated
    # collectives, no kernels waiting on each other).
    backend = os.environ.get("FSTK_BENCH_BACKEND", "nccl")
    if backend != "nccl" and world > 1:
        # several ranks share one GPU here: a per-process device cache could
        # hold memory another rank needs (each can only trim its own).
        os.environ.setdefault("FSTK_DEVICE_CACHE", "0")
    ndev = torch.cuda.device_count()
    local = local % max(ndev, 1) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    import paper_1907_05884_b200 as F
    from paper_1907_05884_b200 import _lib

    model, pts, vals, cfgd = workload(args.config, args.points, rank)
    n = pts.shape[0]
    d = model.order
    fc, fm = flops_per_point(model)
    peak_mma, peak_fma = _lib.fp64_peak(local)

    # ---- device-resident inputs for `value`
    dpts = torch.from_numpy(np.ascontiguousarray(pts.T)).to(dev)  # (d, N): column-major N x d
    # C5 (BASELINE configs[4]): 8 seeded fields sharing one point set, the
    # visualisation stream; every other config evaluates one model.
    models = [model]
    if args.config == "C5":
        from paper_1907_05884_b200 import synth as _s

        models += [_s.random_model(cfgd["ranks"], cfgd["degrees"], cfgd["nnz"], seed=f)
                   for f in range(1, 8)]
    NF = len(models)
    dout = torch.empty((NF, n), dtype=torch.float64, device=dev)

    def eval_step():
        for f, m in enumerate(models):
            m.evaluate_device(dpts, dout[f])

    for _ in range(max(args.warmup, 3)):
        eval_step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    # Between timed steps: inputs larger than L2 need no flush; otherwise a
    # 512 MB buffer is overwritten (outside the per-step event pairs).
    in_bytes = n * d * 8 + n * 8
    flush = None if in_bytes > 2 * L2_BYTES else torch.empty(64 << 20, dtype=torch.float64,
                                                            device=dev)
    launches0 = F.launch_count()
    clocks = Clocks(local)
    _lib.profile_enable(True)
    stream = torch.cuda.current_stream(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    torch.cuda.synchronize()
    for e0, e1 in ev:
        if flush is not None:
            flush.fill_(1.0)
        e0.record(stream)
        eval_step()
        e1.record(stream)
    torch.cuda.synchronize()
    _lib.profile_enable(False)
    ck = clocks.stop()
    launches = F.launch_count() - launches0
    prof = _lib.profile_read()
    ms = sum(e0.elapsed_time(e1) for e0, e1 in ev) / args.steps
    ms = maxreduce(ms, world, dev)
    value = world * n * NF / (ms * 1e-3)

    # ---- roofline of the dominant kernel (the DMMA contraction).  In the
    # timed steps the mode-table kernel of chunk i+1 overlaps the contraction
    # of chunk i on a second stream, so their event durations overlap.  The
    # kernel's own duration comes from an isolated pass of the same chunks on
    # one stream (fstk_gpu_eval_serialize; values unchanged).
    conc = {k: prof[k] for k in ("contract", "mode_tables")}
    iso_steps = 3
    _lib.eval_serialize(True)
    eval_step()
    torch.cuda.synchronize()
    _lib.profile_read()
    _lib.profile_enable(True)
    e_iso = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    e_iso[0].record(stream)
    for _ in range(iso_steps):
        eval_step()
    e_iso[1].record(stream)
    torch.cuda.synchronize()
    _lib.profile_enable(False)
    _lib.eval_serialize(False)
    iso = _lib.profile_read()
    iso_step_ms = e_iso[0].elapsed_time(e_iso[1]) / iso_steps
    c_ms, c_n = iso["contract"]
    m_ms, m_n = iso["mode_tables"]
    assert c_ms / iso_steps <= iso_step_ms * 1.001, "contraction time exceeds its step"
    per_launch_pts = n * NF * iso_steps / max(c_n, 1)
    achieved = fc * n * NF * iso_steps / (c_ms * 1e-3) / 1e12 if c_ms > 0 else None
    traffic, tpts = traffic_from_profile(args.config)
    kr = os.environ.get("FSTK_CONTRACT_KR")
    use_kr = (kr != "0") if kr is not None and model.order in (3, 4) else model.order == 4
    kname = ("contract_kr_kernel (fp64 DMMA m8n8k4, Khatri-Rao K = r0 r1)" if use_kr
             else "contract_kernel (fp64 DMMA m8n8k4)")
    roof = {"bound": "tensor", "kernel": kname,
            "achieved": achieved, "peak": peak_mma, "unit": "TFLOP/s",
            "frac": (achieved / peak_mma) if achieved else None,
            "traffic": (traffic * per_launch_pts / tpts) if traffic and tpts else None,
            "peak_source": "fp64 DMMA throughput measured live on this GPU by fstk_gpu_fp64_peak "
                           "(MEASURED_PEAKS.json has no fp64 entry); DFMA measured %.1f" % peak_fma,
            "algorithmic_flops_per_point": fc,
            "ms_per_launch": c_ms / max(c_n, 1), "launches_per_step": c_n / iso_steps,
            "points_per_launch": per_launch_pts,
            "share_of_step": c_ms / (c_ms + m_ms) if c_ms + m_ms > 0 else None,
            "isolated_step_ms": iso_step_ms,
            "contract_ms_per_step": c_ms / iso_steps,
            "mode_tables_ms_per_step": m_ms / iso_steps,
            "step_tflops": (fc + fm) * n * NF / (ms * 1e-3) / 1e12,
            "step_frac": (fc + fm) * n * NF / (ms * 1e-3) / 1e12 / peak_mma,
            "concurrent_event_ms_per_step": {k: v[0] / args.steps for k, v in conc.items()},
            "note": "achieved/frac: the contraction kernel's algorithmic flops over its own "
                    "event-timed duration in an isolated pass of the same chunks on one stream "
                    "(%d steps). The timed steps overlap it with the next chunk's mode-table "
                    "kernel on a second stream; step_frac is the whole evaluation step "
                    "(all %d flop/pt) at ms_per_step" % (iso_steps, int(fc + fm))}

    # ---- e2e through the host C-ABI (pinned host buffers)
    if NF > 1:
        # C5: the public multi-field call, points uploaded once per step,
        # every field's values read back.
        from paper_1907_05884_b200.model import evaluate_fields

        evaluate_fields(models, pts)
        ef_times = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            evaluate_fields(models, pts)
            ef_times.append(time.perf_counter() - t0)
        ef_s = maxreduce(float(np.median(ef_times)), world, dev)
        e2e = {"value": world * n * NF / ef_s, "unit": UNIT, "h2d_bytes_per_step": int(n * d * 8),
               "d2h_bytes_per_step": int(NF * n * 8), "ms_per_step": ef_s * 1e3,
               "path": "evaluate_fields (pageable numpy points uploaded once, %d fields "
                       "evaluated from HBM through fstk_gpu_evaluate_batch_device, read back)" % NF}
    hp = torch.from_numpy(np.ascontiguousarray(pts.T)).pin_memory()
    hout = torch.empty(n, dtype=torch.float64).pin_memory()
    hp_np = hp.numpy().T  # (N, d) view, column-major
    for _ in range(2):
        model.evaluate_batch_into(hp_np, hout.numpy())
    e2e_times = []
    for _ in range(max(3, min(args.steps, 10))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        model.evaluate_batch_into(hp_np, hout.numpy())
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = maxreduce(float(np.median(e2e_times)), world, dev)
    # Same call with plain (pageable) numpy buffers, as a reference caller
    # passes them: the library stages them through pinned memory.
    pg_times = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        model.evaluate_batch(pts)
        pg_times.append(time.perf_counter() - t0)
    pg_s = maxreduce(float(np.median(pg_times)), world, dev)
    e2e_one = {"value": world * n / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(n * d * 8),
           "d2h_bytes_per_step": int(n * 8), "ms_per_step": e2e_s * 1e3,
           "path": "fstk_gpu_evaluate_batch (host C-ABI), pinned host buffers",
           "pageable": {"value": world * n / pg_s, "ms_per_step": pg_s * 1e3,
                        "path": "the same call with pageable numpy buffers (staged by the "
                                "library through pinned memory)"}}
    if NF == 1:
        e2e = e2e_one
    else:
        e2e["single_field"] = e2e_one

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": DATA_DESC.get(args.config, "synthetic"),
            "config": arm_config(args, model, cfgd, n, NF, world),
            "flops_per_point": fc + fm,
            "roofline": roof, "e2e": e2e, "gpu_launches": int(launches), "clocks": ck}

    # ---- refit (one problem; rows sharded across ranks; one all-reduce)
    if NF > 1 and vals is None and not args.no_refit:
        # C5's fields: seeded tanh fronts with distinct offsets and widths plus
        # Gaussian kernels (BASELINE configs[4]) on the shared points.
        vals = c5_field_values(pts, 0)
    if not args.no_refit and vals is not None:
        # The refit is ONE problem: every rank passes the same (rank-0) cloud.
        rpts, rvals = (pts, vals) if rank == 0 else dataset(args.config, args.points, 0)
        if rvals is None:  # C5 on ranks > 0
            rvals = c5_field_values(rpts, 0)
        line["refit"] = run_refit(model, rpts, rvals, cfgd, args, rank, world, dev, peak_mma)
        if NF > 1 and rank == 0 and world == 1:
            # C5 (BASELINE configs[4]): 8 independent refits with M = 8R each,
            # one per field, on the shared points (each field's values = its
            # model at the points + the config's noise).
            import paper_1907_05884_b200 as F

            per, res = [], []
            R = int(np.prod(model.ranks))
            for f, m in enumerate(models):
                fv = rvals if f == 0 else c5_field_values(rpts, f)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                _, finfo = F.reestimate_core(m, rpts, fv, seed=0, sample_rows=cfgd["m_factor"] * R)
                torch.cuda.synchronize()
                per.append(round(time.perf_counter() - t0, 4))
                res.append(round(finfo["residual_after"], 6))
            line["refit_fields"] = {"fields": NF, "seconds_total": round(sum(per), 4),
                                    "seconds_per_field": per, "residual_after": res,
                                    "sample_rows": cfgd["m_factor"] * R,
                                    "note": "BASELINE C5's 8 independent refits (M = 8R each), "
                                            "sequential on one GPU through reestimate_core"}
        if args.transform != "none" and not args.no_refit_none:
            # The north star's literal estimator (sampled Kronecker rows, no
            # mixing; A never materialised), measured beside the reference's.
            line["refit_none"] = run_refit(model, rpts, rvals, cfgd, args, rank, world, dev,
                                           peak_mma, transform="none")

    if rank == 0 and world == 1 and vals is not None and args.config in ("C1", "C2"):
        line["upstream_idw"] = run_idw(pts, vals, cfgd, args)
    if rank == 0 and not args.no_cpu:
        line["cpu_baseline"] = cpu_eval_baseline(model, pts)
        if vals is not None and not args.no_refit:
            line["cpu_baseline"]["refit"] = cpu_refit_estimate(
                model, pts, vals, cfgd["m_factor"] * int(np.prod(model.ranks)), args.transform)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return 0


def c5_field_values(pts, f: int) -> np.ndarray:
    """Field f of BASELINE configs[4]: a tanh front with its own offset and
    width plus 4 seeded Gaussian kernels, noise sigma 1e-2."""
    rng = np.random.default_rng(700 + f)
    x, y, z = pts[:, 0], pts[:, 1], pts[:, 2]
    off, width = 0.35 + 0.04 * f, 0.015 + 0.004 * f
    v = np.tanh((z - off - 0.05 * np.sin(2 * np.pi * x) * np.sin(2 * np.pi * y)) / width)
    for _ in range(4):
        cx, cy, cz = rng.random(3)
        w, a = rng.uniform(0.02, 0.1), rng.normal(0.0, 0.2)
        v = v + a * np.exp(-((x - cx) ** 2 + (y - cy) ** 2 + (z - cz) ** 2) / (w * w))
    return v + 1e-2 * rng.normal(size=pts.shape[0])


def run_idw(pts, vals, cfgd, args) -> dict:
    """the upstream interpolation of this config's cloud onto its
    grid (C1: 64^3, C2: 256^3; interpolate_to_grid, ingest.cpp:265-383) on the
    GPU through the public call (host arrays in and out), median of three,
    with the oracle restatement on all host cores over a 32^3 sub-grid of the
    same cloud (its index build included) beside it."""
    import paper_1907_05884_b200 as F

    n = 256 if args.config == "C2" else int(cfgd.get("grid", 64))
    pc = F.PointCloud.from_data(pts, vals)
    grid = F.StructuredGrid.unit([n] * pts.shape[1])
    F.interpolate_to_grid(pc, grid)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        _, rep = F.interpolate_to_grid(pc, grid)
        ts.append(time.perf_counter() - t0)
    out = {"nodes": n ** pts.shape[1], "points": int(pts.shape[0]), "seconds": float(np.median(ts)),
           "nodes_per_s": n ** pts.shape[1] / float(np.median(ts)),
           "report": {"box_covered": rep.box_covered, "max_nearest_distance": rep.max_nearest_distance,
                      "extrapolated_fraction": rep.extrapolated_fraction},
           "path": "interpolate_to_grid (fstk_gpu_interpolate_to_grid, host arrays)"}
    if not args.no_cpu:
        from oracle import oracle as O

        t0 = time.perf_counter()
        O.interpolate_to_grid(pts, vals, (32,) * pts.shape[1])
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"seconds_32cubed": dt, "cores": O.max_threads(), "kind": "port",
                               "sample": "the same cloud onto a 32^3 grid (index build included)"}
    return out


def sketch_roofline(model, info, t, transform, world):
    """The sketch (design columns -> DCT/WHT/FFT -> sampled rows) against HBM:
    algorithmic bytes = the mode tables read once + per column the complex
    (real for WHT) q_pad intermediate written and read once between the two
    passes + the S sampled rows written, over this rank's (R+1)/world columns.
    Peak: MEASURED_PEAKS.json hbm_gbs (the driver's copy bandwidth)."""
    if not t or transform == "none":
        return None
    R = int(np.prod(model.ranks))
    q_pad, S = info["padded_rows"], info["sample_rows"]
    elem = 8 if transform == "wht" else 16
    cols = (R + 1) / max(world, 1)
    tables = 8.0 * q_pad * sum(model.ranks)
    per_col = 2.0 * elem * q_pad + 8.0 * S * (2 if transform == "fft" else 1)
    algo = tables + cols * per_col
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak, src = float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        peak, src = 7700.0, "B200_PROFILING.md nominal (MEASURED_PEAKS.json absent)"
    ach = algo / t / 1e9
    return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "algorithmic_bytes": algo, "peak_source": src,
            "kernel": "transform_pass2_kernel (pass 1: design columns + 10 stages; pass 2: 10 "
                      "stages + post-rotation + sampled rows)"}


def gram_roofline(gram_flops, info, t, peak_fp64, i8=None):
    """Gram stage against its roofline.  Native: fp64 SYRK flops vs the DMMA
    peak.  Sliced (fstk_gram.cu): int8 ops issued vs the int8 GEMM ceiling
    measured live on this GPU (int8_peak; MEASURED_PEAKS.json has no int8
    entry), plus the fp64-equivalent rate (R(R+1)S/t) that the DGEMM Gram
    would need to match it."""
    if not t:
        return None
    if info["gram_slices"] > 0 and info.get("gram_int8_ops"):
        ach = info["gram_int8_ops"] / t / 1e12
        pk = i8["tops"] if i8 else 4500.0
        src = i8["source"] if i8 else "nominal B200 dense int8 (live probe unavailable)"
        import paper_1907_05884_b200 as F

        eng = F.gram_engine()
        if eng == "tcgen05":
            kern = (f"syrk_res_kernel (fstk_syrk.cu): hand-written tcgen05.mma.cta_group::2.kind::i8 "
                    f"SYRK, lower-triangle 256x256 tiles, persistent with a dynamic tile scheduler, "
                    f"one launch per column block and CRT modulus, residues reduced in the epilogue; "
                    f"crt_fold4_kernel (Garner) and the residue/exponent kernels in fstk_gram.cu; "
                    f"plane-accuracy level {info['gram_slices']}")
        else:
            kern = (f"cuBLASLt int8 IMMA GEMMs, one per CRT modulus, at plane-accuracy level "
                    f"{info['gram_slices']} (residue/fold kernels in fstk_gram.cu)")
        return {"bound": "tensor", "achieved": ach, "peak": pk, "unit": "TOP/s (int8)",
                "frac": ach / pk, "peak_source": src, "engine": eng,
                "fp64_equivalent_tflops": gram_flops / t / 1e12, "fp64_peak_tflops": peak_fp64,
                "kernel": kern}
    ach = gram_flops / t / 1e12
    return {"bound": "tensor", "achieved": ach, "peak": peak_fp64, "unit": "TFLOP/s",
            "frac": ach / peak_fp64 if peak_fp64 else None,
            "kernel": "cublasDsyrk/Dgemm (library SYRK on the sketched A)"}


def run_refit(model, pts, vals, cfgd, args, rank, world, dev, peak, transform=None):
    import torch

    import paper_1907_05884_b200 as F
    from paper_1907_05884_b200 import synth

    tform = transform or args.transform
    R = int(np.prod(model.ranks))
    S = cfgd["m_factor"] * R
    # Repeated refits of one size: keep the library's large device blocks
    # between sessions (policy 2) unless FSTK_DEVICE_CACHE chose otherwise;
    # the default policy returns them to the driver after every refit.
    from paper_1907_05884_b200 import _lib as _L

    if "FSTK_DEVICE_CACHE" not in os.environ:
        _L.set_device_cache(2)
    # warm-up on a small problem (cuBLAS/cuSOLVER handles, twiddle cache)
    wm = synth.random_model((4, 4, 4), (6, 6, 6), 4, seed=1)
    wp = synth.uniform_points(4096, 3, 2)
    F.reestimate_core(wm, wp, np.sin(wp[:, 0]), seed=1, transform=tform)

    def one():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        sess = F.RefitSession(model, pts, vals, seed=0, sample_rows=S, transform=tform,
                              shard=rank, shards=world, layout="columns" if world > 1 else "rows")
        t_x = 0.0
        if world > 1:
            from paper_1907_05884_b200.dist import exchange_columns

            tx = time.perf_counter()
            exchange_columns(sess)
            t_x = time.perf_counter() - tx
        t_b = time.perf_counter() - t0
        from paper_1907_05884_b200 import _lib as L

        gram = L.device_tensor(R * R, dev)
        rhs = torch.empty(R, dtype=torch.float64, device=dev)
        tn = time.perf_counter()
        sess.normal_equations(gram, rhs)
        torch.cuda.synchronize()
        t_n = time.perf_counter() - tn
        t_ar = 0.0
        if world > 1:
            from paper_1907_05884_b200.dist import reduce_normal_equations

            # ONE all-reduce of the packed lower triangle + rhs.
            ta = time.perf_counter()
            reduce_normal_equations(gram, rhs)
            torch.cuda.synchronize()
            t_ar = time.perf_counter() - ta
        t_hot = time.perf_counter() - t0
        from paper_1907_05884_b200.dist import refine_distributed

        tr = time.perf_counter()
        x = refine_distributed(sess, gram, rhs)
        torch.cuda.synchronize()
        t_r = time.perf_counter() - tr
        tf = time.perf_counter()
        core = sess.finish(x) if rank == 0 else None
        t_f = time.perf_counter() - tf
        t_all = time.perf_counter() - t0
        info = sess.info_dict()
        sess.close()
        del gram
        info["exchange_s"] = t_x
        info["wall_s"] = {"begin": t_b, "normal_equations": t_n, "refine": t_r, "finish": t_f}
        return t_hot, t_all, t_ar, info

    from paper_1907_05884_b200 import _lib

    cold = None
    for _ in range(max(0, args.refit_warmup)):
        c_hot, c_all, _, _ = one()
        cold = cold or {"seconds": c_all, "hot_path_seconds": maxreduce(c_hot, world, dev)}
    # Timed: the median of --refit-reps refits (the int8 Gram and the Cholesky
    # run near the power cap, so single refits vary by ~0.2 s from box to box);
    # then one more with per-kernel event profiling for the stage breakdown.
    reps, rep_stages = [], []
    for _ in range(max(1, args.refit_reps)):
        r_hot, r_all, _, r_info = one()
        reps.append((r_all, maxreduce(r_hot, world, dev)))
        rt, rw = r_info["timings"], r_info["wall_s"]
        rep_stages.append({"prepare": round(rt["prepare_s"], 4), "sketch": round(rt["sketch_s"], 4),
                           "gram": round(rt["gram_s"], 4), "solve": round(rt["solve_s"], 4),
                           "begin_wall": round(rw["begin"], 4), "refine_wall": round(rw["refine"], 4)})
    t_all = float(np.median([r[0] for r in reps]))
    t_hot = float(np.median([r[1] for r in reps]))
    _lib.profile_read()
    _lib.profile_enable(True)
    _, p_all, t_ar, info = one()
    _lib.profile_enable(False)
    kprof = _lib.profile_read()
    tm = info["timings"]
    gram_flops = S / world * R * (R + 1)
    return {"seconds": t_all, "hot_path_seconds": t_hot, "warmup_refits": args.refit_warmup,
            "timed_refits": len(reps), "samples_s": [round(r[0], 4) for r in reps],
            "hot_path_samples_s": [round(r[1], 4) for r in reps], "sample_stages_s": rep_stages,
            "profiled_refit_s": p_all, "cold": cold,
            "scaling": "strong", "sample_rows": S, "working_rows": info["working_rows"],
            "padded_rows": info["padded_rows"], "transform": tform,
            "kernel_ms": {k: v[0] for k, v in kprof.items() if v[1]},
            "kernel_launches": {k: v[1] for k, v in kprof.items() if v[1]},
            "stages_s": {"prepare": tm["prepare_s"], "alloc": tm["alloc_s"], "sketch": tm["sketch_s"],
                         "exchange": info.get("exchange_s", 0.0),
                         "gram": tm["gram_s"], "allreduce": t_ar, "solve": tm["solve_s"],
                         "residual": tm["residual_s"]},
            "host_wall_s": info.get("wall_s"),
            "gram_slices": info["gram_slices"], "refine_steps": info["refine_steps"],
            "gram_roofline": gram_roofline(gram_flops, info, tm["gram_s"], peak,
                                           int8_peak(dev) if info["gram_slices"] > 0 else None),
            "sketch_roofline": sketch_roofline(model, info, tm["sketch_s"], tform, world),
            "residual_before": info["residual_before"], "residual_after": info["residual_after"],
            "rank_deficient": info["rank_deficient"],
            "note": "solve (blocked Cholesky: cuSOLVER diagonal blocks, DTRSM panels, int8 "
                    "tensor-core trailing updates; then refinement against A) is outside the "
                    "hot-path claim (north_star)"}


if __name__ == "__main__":
    sys.exit(main())
