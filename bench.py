#!/usr/bin/env python
"""bench.py -- SRBD MPC solves/s at batch 4096, N=50 (BASELINE.json metric) on B200.

One "step" = one batched pdilqr_step (one SQP/RTI iteration): SRBD linearisation ->
element init -> reverse associative scan -> policy -> forward scan -> dual update -> parallel
filter line search -> in-place update, for B independent instances per GPU.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--batch B] [--N N]
  torchrun --nproc-per-node N bench.py --gpus N ...      (weak scaling: B instances per rank)

Prints ONE JSON line (rank 0).  `value` = instances x steps over all ranks / max-over-ranks device
time of the K timed steps (CUDA events around the stream, barrier + synchronize on both sides).
`e2e` = the same metric through pdilqr_tick_host with pinned HOST buffers (x0 in, u0 + stats out,
copies inside the timed region, one synchronisation per tick).  `roofline` = the dominant kernel's
algorithmic FP32 flops per launch / its average event-timed duration in the timed region, against
the FP32 CUDA-core peak.  `cpu_baseline` = the fp64 C oracle (OpenMP over
instances, all host cores) on a bounded sample of the same workload.  --impl reference times that
oracle as the reference arm.
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

from workloads import synth  # noqa: E402

METRIC = "SRBD MPC solves/s at batch 4096, N=50"
ITER_KEYS = ("x", "u", "lam", "x0", "x_ref", "u_ref", "contact", "feet")
SM_COUNT = 148
FP32_LANES_PER_SM = 128


# ---------------------------------------------------------------------------- flop model
def flops_per_instance(N: int, n: int = 12, m: int = 12, chunk: int | None = None) -> dict:
    """Algorithmic FP32 flops of one step per instance, per kernel (SURVEY
    App. B).  Full combine 16.67 n^3 + 8 n^2, cheap combine (suffix right operand) 8.67 n^3 + 4 n^2,
    element init m^3/3 + 2 m^2 (2n+1) + 6 n^2 m + 4 n m, policy 4 n^2 m + 2 n m^2 + m^3/3 +
    2 m^2 (n+1) + 2 n^2 + 2 n m + (Abar, bbar) 2 n^2 m + 2 n m, forward combine 2 n^3 + 2 n^2,
    forward fold 2 n^2, tail (du, dlam) 2 m n + 2 n^2.  Fused SRBD fold: policy + 4 n^3 + 4 n^2 +
    2 n m + 6 m per stage (no C~, no M solve: X = Abar, DESIGN D7)."""
    L = N + 2
    Lf = N + 1
    c = L if (chunk is None or chunk <= 0) else chunk
    J = -(-L // c)
    Jf = -(-Lf // c)
    full = 16.67 * n ** 3 + 8 * n ** 2
    cheap = 8.67 * n ** 3 + 4 * n ** 2
    # backward: reductions of chunks 1..J-2 (c-1 full each), last chunk folds, tree over J
    # summaries (~J full up-sweep + ~J cheap down-sweep), phase-3 folds of chunks 0..J-2
    if J == 1:
        bwd = (L - 1) * cheap
    else:
        P2 = 1 << (J - 1).bit_length()
        last = L - (J - 1) * c
        bwd = (J - 2) * (c - 1) * full + (last - 1) * cheap + (P2 - 1) * full + (P2 - 1) * cheap + (J - 1) * c * cheap
    if Jf == 1:
        fwd = Lf * 2 * n ** 2
    else:
        P2 = 1 << (Jf - 1).bit_length()
        fwd = (Jf - 1) * (c - 1) * (2 * n ** 3 + 2 * n ** 2) + (P2 - 1) * (2 * n ** 3 + 2 * n ** 2) \
            + Lf * 2 * n ** 2 + (P2 - 1) * 2 * n ** 2
    init = (N + 1) * (m ** 3 / 3 + 2 * m ** 2 * (2 * n + 1) + 6 * n ** 2 * m + 4 * n * m)
    policy = (N + 1) * (4 * n ** 2 * m + 2 * n * m ** 2 + m ** 3 / 3 + 2 * m ** 2 * (n + 1) + 2 * n ** 2 + 2 * n * m
                        + 2 * n ** 2 * m + 2 * n * m)
    tail = (N + 1) * 2 * m * n + (N + 2) * 2 * n ** 2
    # fused single-chunk SRBD path (S = 0, DESIGN D7): policy (incl. Abar, bbar), then the cheap
    # combine with X = Abar: V = P Abar, P' = Q + A^T V (4 n^3), w = p + P b~, p' = Abar^T w + q
    # (4 n^2), b~ = b - B R^-1 r (2 n m + blockwise R^-1 r, 6 m)
    fold_s0 = (N + 1) * (4 * n ** 3 + 4 * n ** 2 + 2 * n * m + 6 * m)
    # the record-fed fold (k_srbd_bwd_fold_r2) skips the structural zeros of the SRBD linearisation:
    # B has nb = 6 nonzero rows (6-11), dt Fx has na = 6 general rows (3-5, 9-11) plus dt at (r, 6 + r),
    # r < 3, so A = I + dt Fx enters H = (P B)^T A and P' = Q + A^T V through na rows; per stage:
    # P B 2 n nb m, G = R + (P B)^T B 2 m nb m, H 2 m na n + 6 m, h = r + (P B)^T b + B^T p 2 n m + 2 nb m,
    # SPD solve m^3/3 + 2 m^2 (n+1), Abar = A + B K 2 nb m n, bbar 2 nb m, V = P Abar 2 n^3,
    # p' = q + Abar^T w 2 n^2, P' 2 na n^2 + 6 n, w = p + P b~ 2 n^2  (the flops it has to do)
    # With the stance compaction the controls of swing feet (zero columns of B) drop out as well:
    # ms = stance controls (6 under the trot of configs 2/3), the count below replaces m by ms in
    # every term that multiplies a column of B or a row of the policy.
    nb = na = 6
    ms = 6

    def fold_count(mm):
        return (N + 1) * (2 * n * nb * mm + 2 * mm * nb * mm + 2 * mm * na * n + 6 * mm + 2 * n * mm + 2 * nb * mm
                          + mm ** 3 / 3 + 2 * mm ** 2 * (n + 1) + 2 * nb * mm * n + 2 * nb * mm + 2 * n ** 3
                          + 2 * n ** 2 + 2 * na * n ** 2 + 6 * n + 2 * n ** 2)
    return {"k_elem_init": init, "k_scan_bwd": bwd, "k_policy": policy, "k_scan_fwd": fwd, "k_tail": tail,
            "k_srbd_bwd_fold": policy + fold_s0, "k_srbd_bwd_fold_struct": fold_count(m),
            "k_srbd_bwd_fold_stance": fold_count(ms),
            "k_srbd_fwd_ls": Lf * 2 * n ** 2 + tail}


def fp32_peak_tflops(sm_mhz: float) -> float:
    return SM_COUNT * FP32_LANES_PER_SM * 2 * sm_mhz * 1e6 / 1e12


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.path = os.path.join("/tmp", f"bench_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "20"], stdout=f, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def _lines(self) -> int:
        try:
            with open(self.path) as f:
                return sum(1 for _ in f)
        except OSError:
            return 0

    def wait_ready(self, timeout: float = 10.0) -> int:
        """Block until nvidia-smi has written its first sample (its start-up takes ~0.1-1 s); return the
        number of lines written so far: samples before the timed region are dropped by stop()."""
        t0 = time.time()
        while self.proc is not None and self._lines() == 0 and time.time() - t0 < timeout:
            time.sleep(0.01)
        return self._lines()

    def stop(self, skip: int = 0) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.03)  # let the sampler flush the last in-region sample
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        for line in list(open(self.path))[skip:]:
            p = [x.strip() for x in line.split(",")]
            if len(p) >= 7:
                rows.append(p)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[3 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------- oracle baseline
def cpu_info() -> dict:
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def cpu_baseline(B: int, N: int, seed: int, budget_s: float = 10.0, sample: int = 1024,
                 latency_horizons=(), lat_budget_s: float = 1.0):
    """The fp64 oracle as it stands (oracle/pdilqr_oracle.c, OpenMP over instances, all host
    cores; built with -march=native on this host) on a bounded sample of the same workload:
    repeated steps of `sample` instances until `budget_s` of wall time.  Plus the single-core p50
    latency of one oracle step (B = 1, config 2) per horizon, each bounded by
    `lat_budget_s`.  Returns solves/s, the latency table and what was run."""
    from oracle import oracle as O
    O.use_native()
    ns = min(sample, B)
    prob = synth.srbd_problem(ns, N=N, seed=seed)
    threads = O.max_threads()
    O.srbd_step(prob, nthreads=threads)
    t0 = time.perf_counter()
    reps = 0
    while True:
        O.srbd_step(prob, nthreads=threads)
        reps += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    lat = {}
    for Nl in latency_horizons:
        p1 = synth.srbd_problem(1, N=Nl, seed=synth.BASE_SEED + 2, randomize=False)
        ts = []
        t1 = time.perf_counter()
        while len(ts) < 3 or (time.perf_counter() - t1 < lat_budget_s and len(ts) < 200):
            q = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in p1.items()}
            a = time.perf_counter()
            O.srbd_step(q, nthreads=1)
            ts.append((time.perf_counter() - a) * 1e6)
        lat[str(Nl)] = {"p50_us": float(np.percentile(ts, 50)), "runs": len(ts)}
    return {"value": ns * reps / dt, "unit": "solves/s", "cores": threads, "kind": "oracle",
            **cpu_info(), "build": O.build_flags(),
            "single_core_latency_us": lat,
            "sample": f"{reps} batched oracle steps of the first {ns} of {B} config-3 instances (N={N}), "
                      f"{dt:.1f} s wall, fp64, {threads} OpenMP threads; latency: one step of config 2 "
                      f"(B=1) on 1 thread per horizon, up to 200 runs or {lat_budget_s:.0f} s"}


def run_reference(args, rank: int):
    if rank != 0:
        return None
    from oracle import oracle as O
    O.use_native()
    ns = min(args.ref_sample, args.batch)
    prob = synth.srbd_problem(ns, N=args.N, seed=synth.BASE_SEED)
    threads = O.max_threads()
    for _ in range(args.warmup):
        O.srbd_step(prob, nthreads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.srbd_step(prob, nthreads=threads)
    dt = time.perf_counter() - t0
    v = ns * args.steps / dt
    sample = f"each step = one batched oracle step of {ns} of the {args.batch} config-3 instances (N={args.N})"
    return {"metric": METRIC, "value": v, "unit": "solves/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (workloads/synth.py, seeded)",
            "config": {"workload": "srbd_mpc_config3", "batch_per_gpu": args.batch, "N": args.N, "n": 12, "m": 12},
            "cpu_baseline": {"value": v, "unit": "solves/s", "cores": threads, "kind": "oracle", "sample": sample,
                             **cpu_info(), "build": O.build_flags()},
            "e2e": {"value": v, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ---------------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=4096, help="instances per GPU (weak scaling)")
    ap.add_argument("--N", type=int, default=50)
    ap.add_argument("--leaf-chunk", type=int, default=0)
    ap.add_argument("--dtype", choices=["f32", "f64"], default="f32")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--ref-sample", type=int, default=256)
    ap.add_argument("--profile-only", action="store_true", help="short run for ncu (no JSON extras)")
    ap.add_argument("--latency", default="25,50,100,200,400,1000",
                    help="horizons of the B=1 latency sweep (config 2), '' to skip")
    ap.add_argument("--latency-reps", type=int, default=1000)
    ap.add_argument("--latency-warmup", type=int, default=50)
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="gloo: CPU collectives (e.g. two ranks sharing one GPU to exercise the sharded path)")
    ap.add_argument("--no-scan-legs", action="store_true", help="skip the B=4096 tree / chunked scan legs")
    ap.add_argument("--gather-out", default="", help="rank 0 saves the gathered [B_total][17] u0 + stats here")
    ap.add_argument("--closed-loop-ticks", type=int, default=50, help="0 disables the closed-loop RTF leg")
    ap.add_argument("--no-large", action="store_true", help="skip the large-dimension LQ leg (configs 4, 5)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        out = run_reference(args, rank)
        if out is not None:
            print(json.dumps(out), flush=True)
        return

    import torch
    import torch.distributed as dist
    import paper_2506_07823_b200 as P
    from paper_2506_07823_b200 import sharding

    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the product path has no CPU fallback)")
    ndev = torch.cuda.device_count()
    local_dev = local % ndev          # ranks may share a device (gloo test runs on a 1-GPU box)
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    coll_dev = dev if args.dist_backend == "nccl" else torch.device("cpu")
    tdt = torch.float32 if args.dtype == "f32" else torch.float64
    B, N = args.batch, args.N

    first, _ = sharding.shard(B, rank)
    prob = synth.srbd_problem(B, N=N, seed=synth.BASE_SEED, first=first)
    h = P.PdIlqr(N=N, n=12, m=12, batch=B, dtype=tdt, model="srbd", srbd=prob["params"],
                 leaf_chunk=args.leaf_chunk, device=local_dev)
    npd = np.float32 if tdt == torch.float32 else np.float64

    def upload():
        return {k: (torch.from_numpy(np.ascontiguousarray(prob[k] if prob[k].dtype == np.uint8 else prob[k].astype(npd)))
                    .to(dev)) for k in ITER_KEYS}

    it = upload()
    stats = h.new_stats()
    stream = torch.cuda.current_stream(dev)

    for _ in range(args.warmup):
        h.step(it, stats)
    torch.cuda.synchronize()
    launches_per_step = h.last_launch_count()
    if args.profile_only:
        for _ in range(args.steps):
            h.step(it, stats)
        torch.cuda.synchronize()
        if rank == 0:
            print(json.dumps({"profile_only": True, "steps": args.steps}), flush=True)
        return

    # --------------------------------------------------------------- timed region (device)
    # No instrumentation inside: the per-kernel breakdown comes from a separate pass below.
    clk = ClockSampler(local_dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk.start()
    skip = clk.wait_ready()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        h.step(it, stats)
    e1.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop(skip)
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    ms_max = sharding.max_over_ranks(ms, world, coll_dev, dist)
    value = world * B * args.steps / (ms_max / 1e3)
    # validation of the timed steps: every instance factorised, finite statistics
    info = stats["info"]
    step_check = {"info_nonzero": int((info != 0).sum().item()), "info_negative": int((info < 0).sum().item()),
                  "theta_finite": bool(torch.isfinite(stats["theta"]).all().item()),
                  "cost_finite": bool(torch.isfinite(stats["cost"]).all().item()),
                  "accepted_last_step": int(stats["accepted"].sum().item())}
    if step_check["info_negative"] or not (step_check["theta_finite"] and step_check["cost_finite"]):
        raise SystemExit(f"bench.py: timed steps produced non-finite results: {step_check}")

    # per-kernel CUDA-event breakdown (separate, untimed pass over the same number of steps)
    h.profile(True)
    for _ in range(min(args.steps, 50)):
        h.step(it, stats)
    torch.cuda.synchronize()
    prof = h.profile_read()
    h.profile(False)

    # final collective (outside the hot path): all-gather of u0 and stats
    gather_ms = None
    gathered = None
    if world > 1:
        packed = sharding.pack_results(it["u"][:, 0, :], stats).to(coll_dev)
        dist.barrier()
        t0 = time.perf_counter()
        if coll_dev.type == "cuda":
            a0 = torch.cuda.Event(enable_timing=True); a1 = torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            gathered = sharding.gather_results(packed, world, dist)
            a1.record(stream)
            torch.cuda.synchronize()
            gather_ms = a0.elapsed_time(a1)
        else:
            gathered = sharding.gather_results(packed, world, dist)
            gather_ms = (time.perf_counter() - t0) * 1e3
    if args.gather_out and rank == 0:
        if gathered is None:   # one rank: its own packed rows (same layout as the gathered tensor)
            gathered = sharding.pack_results(it["u"][:, 0, :], stats)
        torch.save(gathered.cpu(), args.gather_out)

    # --------------------------------------------------------------- e2e via host buffers
    e2e = None
    if not args.no_e2e:
        it = upload()
        x0_host = torch.from_numpy(prob["x0"].astype(npd)).pin_memory()
        u0_host = torch.empty(B, 12, dtype=tdt).pin_memory()
        sh = {"cost": torch.empty(B, dtype=tdt).pin_memory(), "theta": torch.empty(B, dtype=tdt).pin_memory(),
              "alpha": torch.empty(B, dtype=tdt).pin_memory(),
              "accepted": torch.empty(B, dtype=torch.int32).pin_memory(),
              "info": torch.empty(B, dtype=torch.int32).pin_memory()}
        # the public tick (pdilqr_tick_host) captured once into a CUDA graph (PdIlqr.capture_tick_host):
        # every replay copies x0 in from pinned host memory, runs the step and copies u0 + stats out
        tick = h.capture_tick_host(it, x0_host, u0_host, sh)
        for _ in range(args.warmup):
            tick.replay()
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            tick.replay()
            torch.cuda.synchronize()
        e1.record(stream)
        torch.cuda.synchronize()
        t_e2e = sharding.max_over_ranks(e0.elapsed_time(e1), world, coll_dev, dist)
        es = np.dtype(npd).itemsize
        e2e = {"value": world * B * args.steps / (t_e2e / 1e3), "unit": "solves/s",
               "h2d_bytes_per_step": B * 12 * es,
               "d2h_bytes_per_step": B * 12 * es + 3 * B * es + 2 * B * 4,
               "api": "pdilqr_tick_host captured in a CUDA graph (PdIlqr.capture_tick_host): pinned host x0 -> "
                      "step -> host u0 + stats, one replay + device sync per tick"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # --------------------------------------------------------------- roofline of the dominant kernel
    fl = flops_per_instance(N, chunk=h_chunk(args, B, N))
    kern = {k: v for k, v in prof.items() if k in fl}
    dom = max(kern, key=lambda k: kern[k][1]) if kern else None
    sm_mhz = clocks.get("sm_max_mhz") or 1965.0
    peak = fp32_peak_tflops(sm_mhz)
    roof = None
    if dom:
        launches, tot = kern[dom]
        avg_s = tot / launches / 1e3
        ach = fl[dom] * B / avg_s / 1e12
        step_ms = ms / args.steps
        traffic, tsrc = ncu_traffic(dom)
        roof = {"bound": "alu", "kernel": dom, "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                "traffic": traffic, "traffic_unit": "bytes per launch (DRAM read + write)",
                "traffic_source": f"profiles/{tsrc} (ncu --set full, B={B})" if tsrc else None,
                "flops_per_launch": fl[dom] * B, "avg_launch_ms": avg_s * 1e3,
                "share_of_step": (tot / launches) / step_ms,
                "peak_basis": f"FP32 FMA pipe: 148 SMs x 128 lanes x 2 flop x {sm_mhz:.0f} MHz (max SM clock)",
                "per_kernel_ms": {k: v[1] / v[0] for k, v in prof.items()}}
        if dom == "k_srbd_bwd_fold":   # the same time against the flops left after the structural zeros
            roof["flops_basis"] = ("algorithmic: the dense 12x12 D7 Riccati-form count per stage (policy + "
                                   "4n^3 + 4n^2 + 2nm + 6m, DESIGN.md Roofline), the basis of the earlier rounds")
            for key, what in (("k_srbd_bwd_fold_struct", "the products without the structurally zero rows of B "
                               "and the identity part of A"),
                              ("k_srbd_bwd_fold_stance", "as struct, and without the swing-foot controls (zero "
                               "columns of B; 6 stance controls under the trot) -- the flops the kernel has to do")):
                v = fl[key] * B / avg_s / 1e12
                roof[key.replace("k_srbd_bwd_fold_", "count_")] = {"achieved": v, "frac": v / peak,
                                                                   "flops_per_launch": fl[key] * B, "basis": what}
        mp = measured_peaks()
        if mp.get("bf16_tflops"):
            scale = float(mp["bf16_tflops"]) / 2250.0
            roof["peak_measured_scaled"] = peak * scale
            roof["frac_vs_measured_scaled"] = ach / (peak * scale)
            roof["peak_measured_scaled_basis"] = (f"FP32 peak x measured/nominal dense bf16 ({mp['bf16_tflops']:.0f} / "
                                                  f"2250 TFLOP/s, MEASURED_PEAKS.json): no FP32 entry is measured")

    lat = None
    if args.latency:
        lat = latency_sweep(P, torch, dev, [int(v) for v in args.latency.split(",")], args.latency_reps,
                            args.latency_warmup)
    clo = None
    if args.closed_loop_ticks > 0 and args.dtype == "f32":
        clo = closed_loop_bench(P, torch, dev, B, N, args.closed_loop_ticks)
    lq_only = None
    if not args.no_large:
        lq_only = solve_lq_bench(P, torch, dev, h, upload(), B, N, tdt, sm_mhz=(clocks or {}).get("sm_max_mhz") or 1965.0)
    large = None
    if not args.no_large and args.dtype == "f32":
        large = large_bench(P, torch, dev, sm_mhz=(clocks or {}).get("sm_max_mhz") or 1965.0)
    scan_legs = None
    if not args.no_scan_legs and args.dtype == "f32":
        scan_legs = scan_legs_bench(P, torch, dev, B, N, upload, args.steps, peak)
    cpu = None if args.no_cpu_baseline else cpu_baseline(B, N, synth.BASE_SEED, args.cpu_budget,
                                                        latency_horizons=[int(v) for v in args.latency.split(",")]
                                                        if args.latency else [])
    out = {"metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (workloads/synth.py, seeded; config 3)",
           "config": {"workload": "srbd_mpc_config3", "batch_per_gpu": B, "N": N, "n": 12, "m": 12,
                      "leaf_chunk": h_chunk(args, B, N), "n_alpha": 10,
                      "l2": "working set (QP + scan workspace) ~%.2f GB per GPU > 126 MB L2; no flush needed"
                            % (h.workspace.numel() / 1e9),
                      "parallelism": f"batch-sharded dp{world}, no collective on the hot path"
                                     + (f" ({args.dist_backend} for the final gather)" if world > 1 else "")},
           "gpu_launches": launches_per_step * args.steps, "clocks": clocks, "e2e": e2e,
           "roofline": roof, "cpu_baseline": cpu,
           "kernels_ms": {k: v[1] / v[0] for k, v in prof.items()},
           "step_check": step_check, "latency": lat, "scan_legs": scan_legs, "closed_loop": clo,
           "solve_lq_only": lq_only, "large": large}
    if gather_ms is not None:
        out["final_allgather_ms"] = gather_ms
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def latency_sweep(P, torch, dev, horizons, reps, warm=50):
    """Config 2: p50 / p90 single-instance (B=1) pdilqr_step latency vs horizon N, from CUDA-graph
    replays timed one by one with CUDA events (device time), plus the end-to-end tick through
    pdilqr_tick_host (pinned x0 in, u0 + stats out, host synchronisation).  fp32 and fp64."""
    out = {}
    stream = torch.cuda.Stream(dev)
    for dt_name, tdt, npd in (("f32", torch.float32, np.float32), ("f64", torch.float64, np.float64)):
        res = {}
        for N in horizons:
            prob = synth.srbd_problem(1, N=N, seed=synth.BASE_SEED + 2, randomize=False)
            h = P.PdIlqr(N=N, n=12, m=12, batch=1, dtype=tdt, model="srbd", srbd=prob["params"], device=dev.index)
            it = {k: torch.from_numpy(np.ascontiguousarray(prob[k] if prob[k].dtype == np.uint8 else prob[k].astype(npd)))
                  .to(dev) for k in ITER_KEYS}
            st = h.new_stats()
            pristine = {k: it[k].clone() for k in ("x", "u", "lam")}
            with torch.cuda.stream(stream):
                for _ in range(3):
                    h.step(it, st, stream=stream)
                stream.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    h.step(it, st, stream=stream)
                for _ in range(warm):
                    g.replay()
                stream.synchronize()
                ts = []
                for _ in range(reps):
                    for k in ("x", "u", "lam"):      # same input every replay (cold-start iterate)
                        it[k].copy_(pristine[k])
                    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream); g.replay(); e1.record(stream)
                    e1.synchronize()
                    ts.append(e0.elapsed_time(e1) * 1e3)
                # end to end: host x0 -> tick -> host u0 (+ stats), synchronised
                x0h = torch.from_numpy(prob["x0"].astype(npd)).pin_memory()
                u0h = torch.empty(1, 12, dtype=tdt).pin_memory()
                sh = {"cost": torch.empty(1, dtype=tdt).pin_memory(), "theta": torch.empty(1, dtype=tdt).pin_memory(),
                      "alpha": torch.empty(1, dtype=tdt).pin_memory(),
                      "accepted": torch.empty(1, dtype=torch.int32).pin_memory(),
                      "info": torch.empty(1, dtype=torch.int32).pin_memory()}
                te = []
                for r in range(min(reps, 100) + 10):
                    t0 = time.perf_counter()
                    h.tick_host(it, x0h, u0h, sh, stream=stream)
                    stream.synchronize()
                    if r >= 10:
                        te.append((time.perf_counter() - t0) * 1e6)
            res[str(N)] = {"p50_us": float(np.percentile(ts, 50)), "p90_us": float(np.percentile(ts, 90)),
                           "e2e_p50_us": float(np.percentile(te, 50)), "leaf_chunk": 1,
                           "launches": h.last_launch_count()}
            del h, g
        out[dt_name] = res
    return {"metric": "p50 single-solve latency vs horizon N (B=1, config 2, full SQP step)", "unit": "us",
            "timing": "CUDA-graph replay of pdilqr_step, CUDA events per replay (device); e2e = wall time of "
                      "pdilqr_tick_host + stream sync (host)", "per_dtype": out}


def ncu_traffic(kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum (bytes per launch) of `kernel` from the newest
    committed `ncu --set full` summary under profiles/ (r<round>_v<version>_*_ncu.json)."""
    import glob
    import re
    units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    best = None
    for f in glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r*_v*_*ncu.json")):
        m = re.search(r"r(\d+)_v(\d+)_", os.path.basename(f))
        if not m:
            continue
        key = (int(m.group(1)), int(m.group(2)))
        try:
            rows = json.load(open(f))
        except (OSError, ValueError):
            continue
        for r in rows:
            name = r.get("kernel", "").split("<")[0].split()[-1]
            if (name == kernel or name.startswith(kernel + "_r")) and (best is None or key > best[0]):
                tot = 0.0
                for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    v, u = r[k].split()
                    tot += float(v) * units[u]
                best = (key, tot, os.path.basename(f))
    return (best[1], best[2]) if best else (None, None)


def closed_loop_bench(P, torch, dev, B, N, ticks, warm=5):
    """NEXT-1, Table I: B environments, each with its own SRBD MPC,
    one SQP iteration per control tick + RK4 SRBD plant + warm-start shift, all on the GPU.
    Real-time factor = simulated seconds (all envs) per wall second, timed with CUDA events over
    `ticks` ticks; control at 50 Hz (1 node/tick) and 25 Hz (2 nodes/tick, 20 ms nodes)."""
    out = {}
    for k, hz in ((1, 50), (2, 25)):
        L = synth.srbd_problem(B, N + k * (ticks + warm) + 1, seed=synth.BASE_SEED + 7)
        f32 = lambda a: torch.from_numpy(np.ascontiguousarray(a if a.dtype == np.uint8 else a.astype(np.float32))).to(dev)
        h = P.PdIlqr(N=N, n=12, m=12, batch=B, dtype=torch.float32, model="srbd", srbd=L["params"], device=dev.index)
        ref = {key: f32(L[key]) for key in ("x_ref", "u_ref", "contact", "feet")}
        it0 = {"x": f32(L["x"][:, :N + 2]), "u": f32(L["u"][:, :N + 1]), "lam": f32(L["lam"][:, :N + 2])}
        cl = P.ClosedLoop(h, ref, it0, f32(L["x0"]), nodes_per_tick=k)
        for _ in range(warm):
            cl.tick()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(ticks):
            cl.tick()
        e1.record()
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1)
        sim_s = B * ticks * k * float(L["params"]["dt"])
        vref = ref["x_ref"][:, cl.node, 6:8]
        verr = (cl.x_plant[:, 6:8] - vref).abs().mean().item()
        out[f"{hz}hz"] = {"envs": B, "control_hz": hz, "ticks": ticks, "ms_per_tick": ms / ticks,
                          "rtf": sim_s / (ms / 1e3), "rtf_per_env": sim_s / B / (ms / 1e3),
                          "mean_abs_v_err_final": verr,
                          "failed_envs": int((cl.stats["info"] != 0).sum().item())}
        del cl, h
    return {"what": "closed-loop RTI: step + RK4 SRBD plant + shift per node on GPU (fp32, N=%d); rtf = "
                    "simulated env-seconds per wall second (Table I reading R23)" % N,
            "paper_table1_rtf": {"50hz": 370, "25hz": 570, "note": "RTX 3080 + i7-13700KF, JAX + MJX simulator included; context only (P:426-446)"},
            **out}


def ric_flops_per_stage(n: int, m: int) -> float:
    """FP32 flops of one stage of k_big_ric (big_ric.cuh phases 1-6, S present): PB, g, G, H, h,
    Cholesky, two triangular solves per right-hand side (n + 1 of them), Abar, bbar, V, w, P (+ S^T K), p."""
    return (2 * n * n * m + 2 * n * n + 2 * n * m * m + 2 * m * n * n + 2 * n * m + m ** 3 / 3
            + 2 * m * m * (n + 1) + 2 * n * n * m + 2 * n * m + 2 * n ** 3 + 2 * n * n + 2 * n ** 3
            + 2 * n * n * m + 2 * n * n + 4 * n * m)


def solve_lq_bench(P, torch, dev, h_srbd, it, B, N, tdt, sm_mhz, reps=50):
    """pdilqr_solve_lq alone (a2-a6: element init, reverse scan, policy, forward scan,
    du/dlam) on the Eq. 4 data of config 3 -- the SRBD linearisation at the cold-start iterate
    (pdilqr_linearize), solved by a generic LQ handle (n = m = 12, B = 4096, N = 50; single-chunk
    schedule).  CUDA events around `reps` solves, inputs resident."""
    qp = h_srbd.linearize(it)
    qp.pop("info", None)
    h = P.PdIlqr(N=N, n=12, m=12, batch=B, dtype=tdt, device=dev)
    out = h.solve_lq(qp)
    out = h.solve_lq(qp, out=out)
    torch.cuda.synchronize()
    h.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        h.solve_lq(qp, out=out)
    e1.record()
    torch.cuda.synchronize()
    pr = h.profile_read()
    h.profile(False)
    ms = e0.elapsed_time(e1) / reps
    fl = flops_per_instance(N, 12, 12, chunk=N + 2)
    tot = sum(fl[k] for k in ("k_elem_init", "k_scan_bwd", "k_policy", "k_scan_fwd", "k_tail"))
    res = {"what": "pdilqr_solve_lq on the config-3 SRBD linearisation (generic LQ handle, single chunk)",
           "B": B, "N": N, "ms_per_solve_lq": ms, "solves_per_s": B / ms * 1e3,
           "kernels_ms": {k: v[1] / v[0] for k, v in pr.items()}, "info_ok": bool((out["info"] == 0).all()),
           "scan_method_mflop_per_instance": (tot / 1e6) if tot else None,
           "tflops": (tot * B / ms / 1e9) if tot else None,
           "frac_fp32_peak": (tot * B / ms / 1e9 / fp32_peak_tflops(sm_mhz)) if tot else None}
    del h, out, qp
    return res


def large_bench(P, torch, dev, sm_mhz, reps=5):
    """BASELINE configs 4 and 5 on the large-n path.
    Config 4: the centralized controller for 16 quadrupeds (NEXT-3 model, n = m = 192, N = 50;
    workloads.synth.multi_srbd_problem: 16 config-3 robots on a 4 x 4 grid 1.5 m apart, collision
    penalty), one full SQP step (pdilqr_step: multi-robot linearisation, LQ solve, line search,
    update) at B = 1 and B = 64 -- the paper's "< 25 ms for 16 robots" unit (one iteration,
    P:375).  Config 5: pdilqr_solve_lq on the whole-body-sized LQ (n = 74, m = 32, N = 100,
    B = 1024; 4 seeded instances tiled, the kernels' work does not depend on the values).
    CUDA events around `reps` calls (inputs resident; the config-4 iterate restored before each
    step so every rep solves the cold-start problem), per-kernel split from a separate pass."""
    import numpy as np
    res = {}
    keys = ("x", "u", "lam", "x0", "x_ref", "u_ref", "contact", "feet")
    for name, B in (("config4_b1", 1), ("config4_b64", 64)):
        N, R = 50, 16
        prob = synth.multi_srbd_problem(B, R, N=N, seed=synth.BASE_SEED)
        it = {k: torch.from_numpy(np.ascontiguousarray(prob[k] if prob[k].dtype == np.uint8 else prob[k].astype(np.float32)))
              .to(dev) for k in keys}
        pristine = {k: it[k].clone() for k in ("x", "u", "lam")}
        h = P.PdIlqr(N=N, n=12 * R, m=12 * R, batch=B, dtype=torch.float32, model="multi_srbd", srbd=prob["params"],
                     multi=prob["multi"], device=dev)
        st = h.new_stats()
        h.step(it, st)
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            for k in pristine:
                it[k].copy_(pristine[k])
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); h.step(it, st); e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        h.profile(True)
        h.step(it, st)
        torch.cuda.synchronize()
        pr = h.profile_read()
        h.profile(False)
        ms = float(np.median(ts))
        kms = {k: v[1] / v[0] for k, v in pr.items()}
        fl = ric_flops_per_stage(12 * R, 12 * R) * (N + 1) * B
        ric = kms.get("k_big_ric") or kms.get("k_big_ric_tc")
        res[name] = {"B": B, "N": N, "n": 12 * R, "m": 12 * R, "robots": R, "ms_per_step": ms,
                     "solves_per_s": B / ms * 1e3, "kernels_ms": kms, "launches": h.last_launch_count(),
                     "info_ok": bool((st["info"] == 0).all().item()), "alpha": float(st["alpha"][0].item()),
                     "fold_flops": fl, "fold_tflops": (fl / ric / 1e9) if ric else None,
                     "fold_frac_fp32_peak": (fl / ric / 1e9 / fp32_peak_tflops(sm_mhz)) if ric else None,
                     "paper": "< 25 ms per solve for 16 robots on an RTX 3080 (P:18, P:417; context)"}
        del h, it
    for name, B, N, n, m, kind in (("config5_b1024", 1024, 100, 74, 32, "wb"),):
        base = synth.random_lq(min(B, 4), N, n, m, kind=kind, seed=7)
        qp = {}
        for k, v in base.items():
            t = torch.from_numpy(v.astype(np.float32)).to(dev)
            rep = (B + t.shape[0] - 1) // t.shape[0]
            qp[k] = t.repeat((rep,) + (1,) * (t.dim() - 1))[:B].contiguous()
        h = P.PdIlqr(N=N, n=n, m=m, batch=B, dtype=torch.float32, device=dev)
        out = h.solve_lq(qp)
        out = h.solve_lq(qp, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            h.solve_lq(qp, out=out)
        e1.record()
        torch.cuda.synchronize()
        h.profile(True)
        h.solve_lq(qp, out=out)
        torch.cuda.synchronize()
        pr = h.profile_read()
        h.profile(False)
        ms = e0.elapsed_time(e1) / reps
        kms = {k: v[1] / v[0] for k, v in pr.items()}
        fl = ric_flops_per_stage(n, m) * (N + 1) * B
        ric = kms.get("k_big_ric") or kms.get("k_big_ric_tc")
        res[name] = {"B": B, "N": N, "n": n, "m": m, "ms_per_solve_lq": ms, "solves_per_s": B / ms * 1e3,
                     "kernels_ms": kms, "info_ok": bool((out["info"] == 0).all()),
                     "fold_flops": fl, "fold_tflops": (fl / ric / 1e9) if ric else None,
                     "fold_frac_fp32_peak": (fl / ric / 1e9 / fp32_peak_tflops(sm_mhz)) if ric else None}
        del h, out, qp
    return res


def measured_peaks() -> dict:
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


def scan_legs_bench(P, torch, dev, B, N, upload, steps, peak, chunks=(1, 8)):
    """The paper's associative scans at the headline configuration (B = 4096, N = 50): the same
    step with leaf_chunk = 1 (the pure tree of P:195) and an intermediate chunk, instead of the
    single-chunk fold the default picks at B >= 148 (DESIGN D1).  CUDA events around `steps`
    steps (inputs resident); scan-method flops of the flop model / step time vs the FP32 peak."""
    res = {}
    steps = max(5, min(steps, 50))
    prob = synth.srbd_problem(1, N=N)
    for c in chunks:
        h = P.PdIlqr(N=N, n=12, m=12, batch=B, dtype=torch.float32, model="srbd", srbd=prob["params"],
                     leaf_chunk=c, device=dev.index)
        it = upload()
        st = h.new_stats()
        for _ in range(3):
            h.step(it, st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            h.step(it, st)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        h.profile(True)
        for _ in range(5):
            h.step(it, st)
        torch.cuda.synchronize()
        pr = h.profile_read()
        h.profile(False)
        fl = flops_per_instance(N, chunk=c)
        tot = sum(fl[k] for k in ("k_elem_init", "k_scan_bwd", "k_policy", "k_scan_fwd", "k_tail"))
        res[f"leaf_chunk_{c}"] = {"ms_per_step": ms, "solves_per_s": B / ms * 1e3,
                                  "kernels_ms": {k: v[1] / v[0] for k, v in pr.items()},
                                  "scan_method_mflop_per_instance": tot / 1e6,
                                  "frac_fp32_peak": tot * B / ms / 1e9 / peak,
                                  "info_ok": bool((st["info"] == 0).all().item())}
        del h, it, st
    return res


def h_chunk(args, B, N):
    return args.leaf_chunk if args.leaf_chunk > 0 else (N + 2 if B >= 148 else 1)


if __name__ == "__main__":
    main()
