#!/usr/bin/env python
"""Benchmark of the trajectory step -- one JSON line on rank 0.

Default workload: BASELINE.json configs[2] ("c3"): 1d ring L = 16384, N = 8192, Neel
start, projective protocol gamma = 0.3, dt = 0.05, complex128, ONE trajectory.  A "step" is
one full pass of the hot path: U <- K U (dense), Philox clicks + conditional Born sampling +
rank-k projective update, CholeskyQR2.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3|c5|c2|c4]
                    [--mode auto|traj|shard]

N > 1 is launched by the driver with torch.distributed.run (one process per GPU).  With
--mode auto (the default) the single-trajectory configs c3 and c5 are ROW-SHARDED over the N
GPUs (K and U split by rows, NCCL exchange of U fused with the chunked K_g U,
Gram allreduce; strong scaling, BASELINE c3 "single trajectory row-sharded over 1/2/4/8 GPUs"),
with c5 row-sharded as the secondary line; the ensemble configs c1, c2, c4 run
trajectory-parallel (independent trajectories per GPU, no data-path
collective, weak scaling).  At N = 1 both modes are one trajectory on one GPU.
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

import workloads  # noqa: E402

HBM_PEAK_GBS = 6536.7         # MEASURED_PEAKS.json hbm_gbs (copy bandwidth on this pool's B200)
FP64_PEAK_TFLOPS = 37.1        # measured DMMA.8x8x4 issue-rate peak, profiles/r01_fp64_microbench.txt

def _measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


_MP = _measured_peaks()
# INT8 tensor peak: no measured INT8 entry, so the measured bf16 cuBLAS figure x the nominal dense ratio
# 4.5 / 2.25 (B200_PROFILING.md); the sustained figure (power-capped seconds-long loop) for a kernel
# timed inside a long step, the burst one for context
INT8_PEAK_TOPS = 4344.8   # measured tcgen05.mma.kind::i8 issue rate, profiles/r02/int8_peak_microbench.txt
INT8_PEAK_BF16_RATIO = 2.0 * float(_MP.get("bf16_tflops", 1655.2))
INT8_PEAK_SOURCE = ("measured on this pool's B200 (tools/microbench/i8_peak.cu, profiles/r02/int8_peak_microbench.txt): "
                    "back-to-back tcgen05.mma.cta_group::1.kind::i8 128x256x32 on shared-memory-resident random operands, "
                    "148 SMs, best of 3 = 4344.8 TOPS (3806-4345 random, up to 4573 with zero operands; the clock-derived "
                    "8192 MAC/clk/SM x 1965 MHz would be 4766). MEASURED_PEAKS.json has no INT8 entry; its bf16 cuBLAS "
                    f"burst x the nominal 4.5/2.25 ratio gives {INT8_PEAK_BF16_RATIO:.0f}, which this kernel exceeds")
FP64_PEAK_SOURCE = ("measured on this pool's B200: DMMA.8x8x4 microbenchmark 37.1 TF/s (cuBLAS ZGEMM 37.0 TF/s), "
                    "profiles/r01_fp64_microbench.txt; MEASURED_PEAKS.json has no FP64 entry "
                    "(bf16 x 40/2250 nominal ratio would give 29.4)")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", default="c3")
    p.add_argument("--traj-per-gpu", type=int, default=0, help="0: the config's natural batch (1 for c3/c5)")
    p.add_argument("--mode", choices=["auto", "traj", "shard"], default="auto",
                   help="traj: independent trajectories per GPU (weak scaling); shard: one trajectory with K and U "
                        "row-sharded over the GPUs (NCCL exchange + Gram allreduce, strong scaling); auto: shard "
                        "for the single-trajectory configs c3/c5 when N > 1, traj otherwise")
    p.add_argument("--propagator", choices=["dense", "banded"], default="dense",
                   help="dense: the north star's dense K U (default); banded: NEXT-1 stencil passes")
    p.add_argument("--orthonormalizer", choices=["cqr2", "lowrank"], default="cqr2",
                   help="cqr2: CholeskyQR2 (north star); lowrank: NEXT-1 low-rank first pass for the projective step")
    p.add_argument("--protocol", default=None,
                   help="override the config's protocol: projective | homodyne | homodyne_rk4 (NEXT-2) | "
                        "projective_events (NEXT-4)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-fp64-path", action="store_true", help="skip the TRAJ_OZAKI=0 (DMMA) comparison line")
    p.add_argument("--no-observables", action="store_true")
    p.add_argument("--secondary", default="c5",
                   help="also time this config (the metric is quoted at 1d L=16384 and 2d 160x160); 'none' skips")
    p.add_argument("--cpu-budget", type=float, default=120.0, help="seconds of oracle work (reference arm)")
    return p.parse_args()


def workload(args):
    w = workloads.CONFIGS[args.config]()
    if args.protocol:
        import dataclasses
        w = dataclasses.replace(w, protocol=args.protocol)
    # trajectories per GPU as SURVEY §8(d) places them: c3/c5 one (row-shardable); c1 all 16 of
    # the config ("16, batched on 1 GPU"); c2 192 and c4 256 spread over 8 GPUs (24 and 32 each)
    tpg = args.traj_per_gpu or {"c3": 1, "c5": 1, "c1": 16, "c2": 24, "c4": 32}.get(args.config, 8)
    return w, tpg


L2_BYTES = 126e6
OZ_NP = 2   # real INT8 residue products per complex product and modulus (csrc/ozaki.h: the planes re +- j im)


def resolve_mode(args, w, world: int) -> str:
    """auto: row-shard the single-trajectory configs (c3, c5) over N > 1 GPUs, else trajectory-parallel."""
    if args.mode != "auto":
        return args.mode
    return "shard" if world > 1 and w.name in ("c3", "c5") else "traj"


def describe(w, tpg, mode: str = "traj", world: int = 1, args=None):
    proto = f"{w.protocol} gamma={','.join(f'{g:g}' for g in w.gammas)}"
    lat = f"1d ring L={w.L}" if w.Ly == 1 else f"2d torus {w.Lx}x{w.Ly} (L={w.L})"
    place = (f"one trajectory, K and U row-sharded over {world} GPU(s)" if mode == "shard" else
             f"{tpg} trajectory(ies) per GPU")
    d = {"workload": f"{w.name}: {lat}, N={w.N}, {proto}, dt={w.dt}, Neel/checkerboard start, {place}, complex128",
         "L": w.L, "N": w.N, "protocol": w.protocol, "dt": w.dt, "traj_per_gpu": tpg,
         "l2": ("inputs larger than L2 (K is %.2f GB, U %.2f GB per trajectory; L2 = 126 MB)"
                % (16 * w.L * w.L / 1e9, 16 * w.L * w.N / 1e9)
                if 16.0 * w.L * w.L + 32.0 * w.L * w.N * tpg >= L2_BYTES else
                "K and U fit the 126 MB L2: L2 flushed (256 MB write) before every timed call of "
                f"{w.sample_every} steps (the config's sampling interval), per-call CUDA-event times summed"),
         "steps_per_call": w.sample_every,
         "parallelism": (f"row-sharded K,U over {world} GPU(s) (NCCL)" if mode == "shard" and world > 1 else
                         f"trajectory-parallel dp{world}")}
    if args is not None:
        d["propagator"] = args.propagator
        d["orthonormalizer"] = "cqr2" if mode == "shard" else args.orthonormalizer
    return d


# ----------------------------------------------------------------------------- clocks
class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-i", str(self.index), "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [l.split(",") for l in open(self.f.name).read().strip().splitlines() if l.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) >= 8 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 8 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in rows if len(r) >= 8 for j in range(4) if "Active" == r[4 + j].strip()})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


# ----------------------------------------------------------------------------- oracle (CPU)
def cpu_cores() -> int:
    return len(os.sched_getaffinity(0))


def oracle_steps(w, budget_s: float, max_steps: int):
    """Time the oracle (as it stands) on the same workload: one trajectory from the
    Neel state, whole steps, until max_steps or the time budget is used."""
    from threadpoolctl import threadpool_info, threadpool_limits
    from oracle import lattice
    from oracle.trajectory import OracleTrajectory
    # torchrun exports OMP_NUM_THREADS=1; the oracle leg runs alone on rank 0 and gets every core
    # of this process's affinity set
    with threadpool_limits(limits=cpu_cores()):
        K = lattice.propagator_lattice(w.Lx, w.Ly, w.J, w.dt)
        tr = OracleTrajectory(w.Lx, w.Ly, w.protocol, w.gammas[0], w.dt, w.J, seed=w.seed, traj=0, K=K)
        times = []
        t_all = time.perf_counter()
        while len(times) < max_steps:
            t0 = time.perf_counter()
            tr.step(1)
            times.append(time.perf_counter() - t0)
            if time.perf_counter() - t_all > budget_s:
                break
        blas = [f"{i.get('internal_api')} {i.get('version')} x{i.get('num_threads')}" for i in threadpool_info()]
    return times, blas


def cpu_baseline_record(w, budget_s: float, max_steps: int, unit: str):
    times, blas = oracle_steps(w, budget_s, max_steps)
    v = len(times) / sum(times)
    return {"value": v, "unit": unit, "cores": cpu_cores(), "kind": "oracle",
            "sample": f"{len(times)} full oracle step(s) of one {w.name} trajectory from the Neel start "
                      f"(NumPy/SciPy, {'; '.join(blas)}), {sum(times):.1f} s; K construction not timed"}


# ----------------------------------------------------------------------------- our arm
def _dist():
    import torch.distributed as dist
    return dist


def open_handle(P, args, w, mode, rank, world, tpg, stream=None):
    """The handle a user opens for this run: row-sharded (one trajectory, NCCL communicator id
    from rank 0 broadcast over torch.distributed) or a batch of tpg trajectories with global ids
    rank * tpg + t and the folded gamma index of SURVEY §8(d) (workloads.gamma_of)."""
    if mode == "shard":
        uid = None
        if world > 1:
            box = [P.traj_nccl_unique_id() if rank == 0 else None]
            _dist().broadcast_object_list(box, src=0)
            uid = box[0]
        return P.Trajectories(w.Lx, w.Ly, w.protocol, [w.gammas[0]], dt=w.dt, J=w.J, seed=w.seed, traj_base=0,
                              stream=stream, shard_size=world, shard_rank=rank if world > 1 else 0, nccl_id=uid,
                              propagator=args.propagator)
    gam = [w.gamma_of((rank * tpg + t) % w.n_traj) for t in range(tpg)]
    return P.Trajectories(w.Lx, w.Ly, w.protocol, gam, dt=w.dt, J=w.J, seed=w.seed, traj_base=rank * tpg,
                          stream=stream, propagator=args.propagator, orthonormalizer=args.orthonormalizer)


def max_over_ranks(ms: float, world: int) -> float:
    if world == 1:
        return ms
    import torch
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    _dist().all_reduce(t, op=_dist().ReduceOp.MAX)
    return float(t.item())


def run_ours(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # BENCH_SMOKE_ONE_DEVICE=1: launch-logic smoke test of the N > 1 trajectory-parallel path on a
    # one-GPU box (every rank on cuda:0, gloo for the barrier / max-over-ranks); not a measurement
    smoke1 = os.environ.get("BENCH_SMOKE_ONE_DEVICE") == "1"
    if smoke1:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if smoke1:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2508_18468_b200 as P

    w, tpg = workload(args)
    mode = resolve_mode(args, w, world)
    shard = mode == "shard"
    if shard:
        tpg = 1
    tr = open_handle(P, args, w, mode, rank, world, tpg)
    st = tr.stream
    # steps are issued the way a run of the config issues them: one traj_step call per interval
    # between sampled observables (w.sample_every steps; the fused small-lattice path runs a call
    # as one launch, the general path as its per-step launches)
    def run_steps(n):
        done = 0
        while done < n:
            k = min(max(1, w.sample_every), n - done)
            tr.step(k)
            done += k
    run_steps(args.warmup)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    tr.profile(True)
    clocks = Clocks(local)
    clocks.start()
    l0 = P.traj_kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    fits_l2 = 16.0 * w.L * w.L + 32.0 * w.L * w.N * tpg < L2_BYTES
    if fits_l2:
        # K and U fit the L2: flush it (a 256 MB write) before every timed call, outside the
        # event pair, and sum the per-call device times
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        ms, done = 0.0, 0
        while done < args.steps:
            k = min(max(1, w.sample_every), args.steps - done)
            flush.fill_(done & 0xff)
            torch.cuda.synchronize()
            e0.record(st)
            tr.step(k)
            e1.record(st)
            torch.cuda.synchronize()
            ms += e0.elapsed_time(e1)
            done += k
        del flush
    else:
        e0.record(st)
        run_steps(args.steps)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    if world > 1:
        dist.barrier()
    launches = P.traj_kernel_launches() - l0
    clk = clocks.stop()
    phases = tr.phase_times()
    tr_clicks = ([tr.last_clicks(t) for t in range(tpg)]
                 if w.protocol in ("projective", "projective_events") else [(0, 0)])
    ms_max = max_over_ranks(ms, world)
    value = (1 if shard else world) * tpg * args.steps / (ms_max / 1e3)
    rows = w.L // world if shard else w.L
    oz = tr.ozaki_info()
    roof, executed, hbm, library = roofline(args, w, tpg, shard, rows, phases, tr_clicks, ms, P, oz)
    # ---- row a4, timed separately (north star: "eigvalsh on C_A at sampled times, timed
    # separately"): the config's sampled observables once, after the timed steps
    obs = None
    if not args.no_observables:
        obs = {}
        for name, region in w.regions.items():
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if isinstance(region, tuple):
                tr.mutual_info(*region)
                kind = "I2"
            else:
                tr.entropy(region)
                kind = "S_A"
            obs[f"{kind}:{name}"] = 1e3 * (time.perf_counter() - t0)
    tr.close()
    del tr
    # the workspace block stays in torch's caching allocator, so the e2e handle below takes it from
    # there as a user's next handle would (a fresh 29 GB cudaMalloc after a free costs ~0.4 s)

    # ---- the same step on the FP64 tensor pipe (TRAJ_OZAKI=0: the DMMA kernels), for the metric's
    # "FP64 tensor TFLOP/s vs peak" read literally: executed DMMA flops of its dominant phase over that
    # phase's device time against the measured 37.1 TF/s DMMA peak
    fp64_path = None
    if oz[0] and not shard and world == 1 and not args.no_fp64_path:
        torch.cuda.empty_cache()
        fp64_path = run_fp64_path(args, w, tpg, P)

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, w, tpg, mode, rank, world, P)

    # ---- the metric's second lattice (2d 160x160), same step, same timing rules, same mode
    secondary = None
    if args.secondary and args.secondary not in ("none", '""', "''") and args.secondary != args.config:
        torch.cuda.empty_cache()
        secondary = run_secondary(args, world, rank, P)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    out = {
        "metric": "trajectory steps/s (configs[2]: 1d L=16384 projective; metric also quoted at 2d 160x160)",
        "value": value, "unit": "trajectory-steps/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "strong" if shard else "weak",
        "vs_baseline": None,
        "dtype": dtype_of(oz), "data": "synthetic (Neel start, Philox randoms, seed 0)",
        "config": describe(w, tpg, mode, world, args),
        "roofline": roof,
        "step_executed": executed,
        "library_same_shape": library,
        "hbm_kernels": hbm or None,
        "phases_ms_per_step": {k: v[0] / args.steps for k, v in phases.items()},
        "phases_nested": {"ku_mma": "propagate", "gram_mma": "gram", "trmm_mma": "trmm",
                          "struct_factor": "chol"},
        "phase_launches_per_step": {k: v[1] / args.steps for k, v in phases.items()},
        "gpu_launches": launches,
        "sampled_observables_ms": obs,
        "secondary": secondary,
        "fp64_tensor_path": fp64_path,
        "clocks": clk,
        "e2e": e2e,
    }
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline_record(w, budget_s=20.0, max_steps=1, unit="trajectory-steps/s")
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def strassen_levels(w, P: int = 1, T: int = 1) -> int:
    """Strassen levels of the planar K U (the rule of csrc/traj_api.cu carve(); row-sharded over P GPUs:
    csrc/shard.cu's rule on the Lp x Lp chunks K_g[:, s], Lp = L / P, at most two levels)."""
    Lp = w.L // P
    if (os.environ.get("TRAJ_STRASSEN", "1") == "0" or Lp % 2 or w.N % 2
            or w.N < int(os.environ.get("TRAJ_STRASSEN_MIN_N", "2048"))):
        return 0
    r16 = lambda x: (x + 15) // 16 * 16
    two_ok = Lp % 4 == 0 and w.N % 4 == 0 and 147.0 * P * (Lp // 4) * r16(Lp // 4) * 8 <= 24e9
    three_ok = P == 1 and T == 1 and w.L % 16 == 0 and 1029.0 * (w.L // 8) * r16(w.L // 8) * 8 <= 40e9
    want = int(os.environ.get("TRAJ_STRASSEN_LEVELS", "3"))
    return 3 if want >= 3 and three_ok else (2 if want >= 2 and two_ok else 1)


def dtype_of(oz):
    if oz and (oz[0] or oz[1]):
        parts = [x for x, on in (("K U", oz[0]), ("the CholeskyQR Grams / TRMMs", oz[1])) if on]
        return (f"c128 (FP64 values; {' and '.join(parts)} as exact modular products on the INT8 tensor cores, "
                f"{oz[2]} moduli with a square root of -1 each = two real residue products per complex product and "
                f"{ {16: 57, 18: 61}.get(oz[2], '?') }-bit operand rows/columns, CRT to FP64; the rest FP64 on DMMA / FP64 "
                "pipes)")
    return "c128 (f64 arithmetic)"


def roofline(args, w, tpg, shard, rows, phases, tr_clicks, ms, P, oz=(False, False, 0)):
    """Roofline of the dominant phase (the largest device time per step) on EXECUTED flops.

    Work per step in conventional 8mnk complex flops, per GPU (rows = L/P of the
    L rows when row-sharded):
      propagate (dense K U): 8 rows L N
      gram (G = U^dag U, upper tiles): 4 rows N^2 per measured Gram -- one per projective step
        (pass 1's Gram comes from the zeroed rows), two otherwise
      trmm (U <- U R^-1): 4 rows N^2 per TRMM counted in this phase -- the second pass only when
        the first is overlapped with the Cholesky (its time is then in the chol phase)
    The 3M (Gauss) schemes -- the planar real products and the interleaved zgemm3m kernels -- issue
    6mnk flops on the DMMA pipe for every 8mnk: `achieved` / `frac` count those executed flops;
    `achieved_8mnk_equiv` / `frac_8mnk_equiv` state the conventional-count equivalent."""
    algo = P.traj_get_zgemm_algorithm()
    kn = {"3m": ("zgemm3mw_dmma_kernel<0,0> (3M, 128x64 CTA)", "zgemm3m_dmma_kernel<1,0> (3M, 64x64 CTA)"),
          "4m": ("zgemm_dmma_kernel<0,0> (4M)", "zgemm_dmma_kernel<1,0> (4M)")}[algo]
    plan_on = os.environ.get("TRAJ_PLANAR_MIN_N")
    big = w.N >= (int(plan_on) if plan_on else 512)
    planar = (args.propagator == "dense" and big and os.environ.get("TRAJ_PLANAR_KU", "1") != "0"
              and w.protocol in ("projective", "homodyne")
              and (not shard or os.environ.get("TRAJ_PLANAR_CQR", "1") != "0"))
    planar_cqr = big and os.environ.get("TRAJ_PLANAR_CQR", "1") != "0" and (not shard or planar)
    slv = strassen_levels(w, w.L // rows, tpg) if planar else 0
    strassen = slv > 0
    ku_name = (f"dgemm_dmma_kernel x{3 * 7 ** slv} (planar 3M: Kr Ur, Ki Ui, (Kr+Ki)(Ur+Ui), each by {slv} "
               f"Strassen level(s): {7 ** slv} products of 1/{2 ** slv} size; 128x128 CTA, one batched launch) + "
               "operand / recombination passes"
               if strassen else
               "dgemm_dmma_kernel x3 (planar 3M: Kr Ur, Ki Ui, (Kr+Ki)(Ur+Ui); 128x128 CTA) + split/combine passes"
               + ("; per shard: P ring-distance K-chunk products accumulated, the U exchange under them" if shard
                  else "")
               if planar else kn[0])
    gram_name = ("dgemm_dmma_kernel<1> x3 (planar 3M: Ur^T Ur, Ui^T Ui, (Ur-Ui)^T (Ur+Ui); upper tiles) + split/combine"
                 if planar_cqr else f"{kn[1]}: G = U^dag U upper tiles")
    trmm_name = ("dgemm_dmma_kernel<0> x3 (planar 3M against X's planes, triangle skipped) + split/combine"
                 if planar_cqr else f"{kn[0]} triangular")
    n_gram = 1 if (w.protocol == "projective" and os.environ.get("TRAJ_LOWRANK_GRAM", "1") != "0") else 2
    nS0 = sum(c[0] for c in tr_clicks) / max(1, tpg)
    struct0 = (w.protocol == "projective" and args.orthonormalizer == "cqr2" and 0 < 2 * nS0 <= w.N
               and os.environ.get("TRAJ_STRUCT_CHOL", "1") != "0")
    # the TRMMs timed in the trmm phase: pass 2's; pass 1's too unless it ran inside the chol phase
    # (overlapped with the factorisation, or the structured pass 1)
    n_trmm = 1 if (struct0 or os.environ.get("TRAJ_CHOL_OVERLAP", "1") != "0") else 2
    # DMMA flops per 8mnk flop: 3M 6/8; with one Strassen level 7/8 of that (21 half-size products)
    a_ku = 0.75 * (7 / 8) ** slv if (planar or algo == "3m") else 1.0
    a_cqr = 0.75 if (planar_cqr or algo == "3m") else 1.0
    kern = {"propagate": (8.0 * rows * w.L * w.N * tpg, a_ku, f"{ku_name}: U <- K U (8 L^2 N flops per step)"),
            "gram": (n_gram * 4.0 * rows * w.N * w.N * tpg, a_cqr,
                     f"{gram_name}: {n_gram} measured Gram(s) per step, 4 L N^2 each"),
            "trmm": (n_trmm * 4.0 * rows * w.N * w.N * tpg, a_cqr,
                     f"{trmm_name}: U <- U R^-1, {n_trmm} TRMM(s) in this phase per step, 4 L N^2 each")}
    if args.propagator == "banded":
        kern.pop("propagate")
    k_sum = sum(c[0] for c in tr_clicks)
    k1_sum = sum(c[1] for c in tr_clicks)
    if args.orthonormalizer == "lowrank" and w.protocol == "projective" and not shard:
        # no N x N Gram / TRMM per step: the work is the four rank-k GEMMs of the projective phase,
        # 16 L N (k1 + k0) flops per trajectory (U W, U -= T W^dag, U' V^dag, U' += P F V); k from
        # the last timed step's clicks; the phase time also holds the sampler and Newton-Schulz
        kern = {"project": (16.0 * w.L * w.N * k_sum, 1.0 if algo == "4m" else 0.75,
                            f"projective rank-k GEMMs ({kn[1].split(' ')[0].split('<')[0]} family): 16 L N (k1 + k0) "
                            f"flops per step, k1 + k0 = {k_sum} clicks in the last timed step; phase time includes "
                            "the blocked sampler and the Newton-Schulz iteration")}
    fused = phases.get("fused", (0.0,))[0] > 0
    if fused:
        # the fused small-lattice step (small_step.cu): the whole step in one CTA per trajectory,
        # 4M complex tiles as four real m8n8k4 DMMAs; algorithmic flops per trajectory-step
        # 8 L^2 N (K U) + 2 x (4 L N^2 Gram + 4 L N^2 solve)
        kern = {"fused": ((8.0 * w.L * w.L * w.N + 16.0 * w.L * w.N * w.N) * tpg, 1.0,
                          "small_step_kernel: the whole step (K U, monitor, CholeskyQR2) with U in shared "
                          "memory, one CTA per trajectory, 4M complex tiles on DMMA m8n8k4; "
                          "8 L^2 N + 16 L N^2 flops per trajectory-step")}
    dom = max(kern, key=lambda k: phases[k][0])
    kern_ms = phases[dom][0] / args.steps
    flops8, alpha, kname = kern[dom]
    eq8 = flops8 / (kern_ms / 1e3) / 1e12
    achieved = eq8 * alpha
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp) and dom == "propagate" and not shard:
        try:
            tj = json.load(open(tp)).get(w.name, {})
            traffic = (tj.get(f"propagate_strassen{slv}_dram_bytes") if strassen else
                       tj.get("propagate_dram_bytes") if planar else tj.get("interleaved_zgemm3mw_dram_bytes"))
        except Exception:
            traffic = None
    mult = (f"planar 3m + {slv} Strassen level(s)" if (strassen and dom == "propagate") else
            "planar 3m" if (planar and dom == "propagate") or (planar_cqr and dom in ("gram", "trmm")) else
            "4m" if dom == "fused" else algo)
    roof = {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
            "achieved_8mnk_equiv": eq8, "frac_8mnk_equiv": eq8 / FP64_PEAK_TFLOPS,
            "kernel": kname + ("; per shard (L/P rows) when row-sharded" if shard else ""),
            "kernel_ms": kern_ms, "timed": "device time of that phase per step (CUDA events around it on "
                                          "the handle's stream)", "peak_source": FP64_PEAK_SOURCE,
            "complex_mult": mult,
            "flops_counted": ("executed DMMA flops: 6mnk per complex product for 3M (three real products), "
                              "x 7/8 per Strassen level on each real product (seven products of half size), 8mnk "
                              "for 4M; achieved_8mnk_equiv counts the conventional 8mnk"),
            "traffic_note": (("ncu dram bytes of the propagate phase (profiles/ncu_traffic.json: U's Strassen "
                              f"operands, the {3 * 7 ** slv} real products as one batched launch, the "
                              "recombination) vs 8.6 GB algorithmic") if strassen else
                             ("ncu dram bytes of the propagate phase (profiles/ncu_traffic.json: split, the "
                              "three real 16384x8192x16384 products as one batch-3 launch, combine) vs 8.6 GB "
                              "algorithmic")) if traffic else None}
    oz_dom = (oz[0] and dom == "propagate") or (oz[1] and dom in ("gram", "trmm"))
    # (a dominant Gram / TRMM phase whose modular launch never ran — e.g. the event-driven step's dense
    # CholeskyQR below the modular size — keeps the DMMA roofline above)
    oz_dom = oz_dom and phases.get({"propagate": "ku_mma", "gram": "gram_mma", "trmm": "trmm_mma"}[dom], (0.0,))[0] > 0
    if oz_dom:
        # the dominant phase is an exact modular product (csrc/ozaki.h): 2 s INT8 products per complex
        # product (the two planes re +- j im of each of the s moduli); algorithmic INT8 ops (2 per MAC) over the nested
        # phase that times the INT8 tensor-core launch alone; its phase time adds the residue
        # splits and the CRT combine
        s_ = oz[2]
        mma_ph = {"propagate": "ku_mma", "gram": "gram_mma", "trmm": "trmm_mma"}[dom]
        mma_ms = phases[mma_ph][0] / args.steps
        per = {"propagate": 2.0 * OZ_NP * s_ * rows * w.L * w.N * tpg,
               "gram": n_gram * 2.0 * OZ_NP * s_ * (w.N * w.N / 2.0) * rows * tpg,
               "trmm": n_trmm * 2.0 * OZ_NP * s_ * rows * (w.N * w.N / 2.0) * tpg}[dom]
        tops = per / (mma_ms / 1e3) / 1e12
        eqp = flops8 / (kern_ms / 1e3) / 1e12
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        traffic = None
        if os.path.exists(tp) and dom == "propagate":
            try:
                traffic = json.load(open(tp)).get(w.name, {}).get(f"ku_ozaki{s_}_igemm_dram_bytes")
            except Exception:
                traffic = None
        roof = {"bound": "tensor", "achieved": tops, "peak": INT8_PEAK_TOPS, "unit": "TOPS (INT8)",
                "frac": tops / INT8_PEAK_TOPS, "traffic": traffic,
                "kernel": ("igemm_i8_kernel (tcgen05.mma.kind::i8, TMEM accumulators, TMA 128B-swizzled K-major "
                           f"tiles, 128x256x128 CTA tile, persistent): one launch of the {OZ_NP} x {s_} residue products "
                           + {"propagate": "of U <- K U (K's residues formed once)",
                              "gram": "of G = U^dag U (upper tiles)",
                              "trmm": "of U <- U R^-1 (triangular k-blocks skipped)"}[dom]
                           + ("; per shard (L/P rows): the P ring-ordered K-chunk products K_g[:, s] U_s, their "
                              "residues accumulated in the epilogue, one CRT combine" if shard and dom == "propagate"
                              else "; per shard (L/P rows)" if shard else "")),
                "kernel_ms": mma_ms, "timed": ("device time of the INT8 launch per step (CUDA events around it on "
                                                "the handle's stream, nested phase " + mma_ph + ")"),
                "ops_counted": (f"2 x {OZ_NP} x {s_} x (the complex product's m n k; half for the Gram's and TRMM's "
                                "triangles) INT8 multiply-adds: algorithmic, tile waste not counted"),
                "peak_source": INT8_PEAK_SOURCE,
                "phase_ms": kern_ms, "phase_note": "the phase adds U's residue split and the CRT combine",
                "fp64_equiv_tflops": eqp, "fp64_equiv_frac_of_dmma_peak": eqp / FP64_PEAK_TFLOPS,
                "fp64_equiv_note": (f"conventional 8mnk complex flops of the phase over its whole time, against the "
                                    f"{FP64_PEAK_TFLOPS} TF/s DMMA peak: an equivalent, not a pipe fraction")}
    if w.name == "c1":
        roof["note"] = ("c1 is latency-bound (SURVEY §8(d)): L = 64, one fused launch per step with one CTA per "
                        "trajectory, whose ~140 barriers and dependent pivots set the time; the fraction is not a "
                        "kernel-quality figure")
    # executed DMMA flops of the whole step (model of what the kernels issue), over the step time
    k1 = k1_sum / max(1, tpg)
    nS = k_sum / max(1, tpg)
    k0 = nS - k1
    a3 = 0.75 if algo == "3m" else 1.0
    structured = (w.protocol == "projective" and args.orthonormalizer == "cqr2" and k0 > 0
                  and os.environ.get("TRAJ_STRUCT_CHOL", "1") != "0" and 2 * nS <= w.N)
    sb = int(os.environ.get("TRAJ_STRUCT_B", "128"))
    step8 = {"propagate": (8.0 * rows * w.L * w.N if args.propagator == "dense" else 0.0, a_ku),
             "gram": (n_gram * 4.0 * rows * w.N * w.N, a_cqr),
             "project": (16.0 * rows * w.N * k1 + 8.0 * nS * nS * w.N if w.protocol == "projective" else 0.0, a3)}
    if structured:
        # pass 1 on the structure of I - V^dag V (csrc/structchol.cu): the factorisation
        # 24 k0^2 N + 8 b k0 N + (8/3) b^2 N, the solve 16 L N k0 + 4 L N b; pass 2 measured Gram + TRMM
        step8["chol"] = (24.0 * k0 * k0 * w.N + 8.0 * sb * k0 * w.N + (8.0 / 3.0) * sb * sb * w.N
                         + 16.0 * rows * w.N * k0 + 4.0 * rows * w.N * sb, a3)
        step8["trmm"] = (4.0 * rows * w.N * w.N, a_cqr)
    else:
        step8["chol"] = ((8.0 / 3.0) * w.N ** 3, a3)
        step8["trmm"] = (2 * 4.0 * rows * w.N * w.N, a_cqr)
    executed = None
    if not fused and not (args.orthonormalizer == "lowrank" and w.protocol == "projective" and not shard) \
            and w.protocol in ("projective", "homodyne"):
        # phases on the INT8 modular path leave the DMMA sum: their INT8 ops are counted apart
        int8_ph = ({"propagate"} if oz[0] else set()) | ({"gram", "trmm"} if oz[1] else set())
        i8 = sum(OZ_NP * oz[2] * 2.0 * (step8[k][0] / 8.0) for k in int8_ph)   # 8mnk / 8 = complex MACs
        fl = sum(f * a for k, (f, a) in step8.items() if k not in int8_ph) * tpg
        i8 *= tpg
        t = ms / args.steps / 1e3
        executed = {"tflops": fl / t / 1e12, "frac": fl / t / 1e12 / FP64_PEAK_TFLOPS, "flops_per_step": fl,
                    "engine_note": ("tflops / frac: DMMA (FP64 tensor pipe) flops of the phases still on it, over the "
                                    "whole step time" + ("; int8_*: the modular products' INT8 ops (2 x 2 s per "
                                                         "complex m n k) over the whole step time" if int8_ph else "")),
                    "int8_phases": sorted(int8_ph),
                    "int8_ops_per_step": i8 or None, "int8_tops": (i8 / t / 1e12) if i8 else None,
                    "model": ("per step (and per shard, rows = L/P): K U 8 rows L N; the measured Gram(s) 4 rows N^2; "
                              "the projective update 16 rows N k1 + C_SS 8 |S|^2 N; " +
                              ("CholeskyQR pass 1 on the structure of I - V^dag V (k0 = |S| - k1 zeroed rows, "
                               f"column blocks b = {sb}): 24 k0^2 N + 8 b k0 N + (8/3) b^2 N + 16 rows N k0 + "
                               "4 rows N b, pass 2's TRMM 4 rows N^2" if structured else
                               "one chol_inverse (8/3) N^3 (the second CholeskyQR pass takes the first-order "
                               "factor), two TRMMs 4 rows N^2") +
                              "; each x 0.75 for the 3M schemes (the DMMA flops they issue)"),
                    "structured_pass1": structured, "k1": k1, "k0": k0,
                    "per_phase_8mnk": {k: v[0] * tpg for k, v in step8.items()}}
    # same-shape library denominators (tools/library_compare.py, committed under profiles/):
    # cublasZgemm / cublasZgemm3m for K U, cuSOLVER potrf + trtri for the Cholesky inverse
    library = None
    lp = os.path.join(ROOT, "profiles", "r01", f"library_compare_{w.name}.json")
    if os.path.exists(lp) and not shard and args.propagator == "dense":
        try:
            lc = json.load(open(lp))
            library = {"source": os.path.relpath(lp, ROOT) + " (tools/library_compare.py, same shapes, same box type)",
                       "K_U_ms": {k: round(v["ms"], 2) for k, v in lc["K_U"].items()},
                       "K_U_note": "ours_planar_3x_dgemm is the three real products the propagator launches "
                                   "(its split/combine passes add about 1.5 ms)",
                       "chol_inverse_ms": {k: round(v["ms"], 2) for k, v in lc["chol_inverse"].items()
                                           if isinstance(v, dict)}}
        except Exception:
            library = None
    # HBM-bound kernels of the step (a2 homodyne "32 L N bytes"; NEXT-1 banded stencil
    # 32 L N bytes per 1d pass, two passes in 2d): algorithmic bytes / event-timed phase time
    hbm = {}
    if w.protocol == "homodyne" and phases["monitor"][0] > 0:
        b = 32.0 * rows * w.N * tpg * args.steps
        g = b / (phases["monitor"][0] / 1e3) / 1e9
        hbm["row_monitor_kernel (homodyne, 32 L N B/step)"] = {
            "achieved_gbs": g, "peak_gbs": HBM_PEAK_GBS, "frac": g / HBM_PEAK_GBS,
            "ms_per_step": phases["monitor"][0] / args.steps,
            "note": "algorithmic bytes over the phase time; the monitor reads U right after the propagate "
                    "wrote it, so up to the 126 MB L2's worth comes from L2 (frac can exceed 1 when U is a "
                    "few L2s, as at c4)"}
    if args.propagator == "banded" and phases["propagate"][0] > 0:
        passes = 1 if w.Ly == 1 else 2
        b = 32.0 * passes * rows * w.N * tpg * args.steps
        g = b / (phases["propagate"][0] / 1e3) / 1e9
        hbm[f"banded_kernel ({passes} pass(es), 32 L N B each)"] = {"achieved_gbs": g, "peak_gbs": HBM_PEAK_GBS,
                                                                   "frac": g / HBM_PEAK_GBS,
                                                                   "ms_per_step": phases["propagate"][0] / args.steps}
    if w.protocol == "projective_events" and phases["project"][0] > 0:
        # one pass per event reads U once and writes it once (32 L N bytes); events of the last window
        b = 32.0 * w.L * w.N * k_sum * args.steps
        g = b / (phases["project"][0] / 1e3) / 1e9
        hbm["ev_pass_1d_kernel (one pass per event, 32 L N B; events in the last window)"] = {
            "achieved_gbs": g, "peak_gbs": HBM_PEAK_GBS, "frac": g / HBM_PEAK_GBS,
            "ms_per_step": phases["project"][0] / args.steps}
    if w.protocol == "homodyne_rk4" and phases["propagate"][0] > 0:
        b = 4 * 48.0 * rows * w.N * tpg * args.steps
        g = b / (phases["propagate"][0] / 1e3) / 1e9
        hbm["horner_pass_kernel (RK4 as 4 Horner passes, 48 L N B each)"] = {
            "achieved_gbs": g, "peak_gbs": HBM_PEAK_GBS, "frac": g / HBM_PEAK_GBS,
            "ms_per_step": phases["propagate"][0] / args.steps}
    ev_key = next((k for k in hbm if k.startswith("ev_pass")), None)
    if w.protocol == "projective_events" and args.orthonormalizer == "lowrank" and ev_key:
        # the event-driven step with the probe certificate is one HBM read + write of U per event
        roof = {"bound": "hbm", "achieved": hbm[ev_key]["achieved_gbs"], "peak": HBM_PEAK_GBS, "unit": "GB/s",
                "frac": hbm[ev_key]["frac"], "traffic": None, "kernel": ev_key,
                "kernel_ms": hbm[ev_key]["ms_per_step"], "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    return roof, executed, hbm, library


def run_secondary(args, world, rank, P, steps=2, warmup=2):
    """Time the secondary config (default c5: 2d 160x160 projective) with the same step, the
    same propagator/orthonormaliser, the same mode (row-sharded over the N GPUs when the primary
    is) and CUDA events; max over ranks."""
    import torch
    import dataclasses
    w = workloads.CONFIGS[args.secondary]()
    if args.protocol:
        w = dataclasses.replace(w, protocol=args.protocol)
    mode = resolve_mode(args, w, world)
    tr = open_handle(P, args, w, mode, rank, world, 1)
    for _ in range(warmup):
        tr.step(1)
    torch.cuda.synchronize()
    if world > 1:
        _dist().barrier()
    tr.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(tr.stream)
    for _ in range(steps):
        tr.step(1)
    e1.record(tr.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ph = tr.phase_times()
    tr.close()
    del tr
    torch.cuda.empty_cache()
    ms = max_over_ranks(ms, world)
    shard = mode == "shard"
    rows = w.L // world if shard else w.L
    prop = ph["propagate"][0] / steps
    out = {"config": describe(w, 1, mode, world, args), "value": (1 if shard else world) * steps / (ms / 1e3),
           "unit": "trajectory-steps/s", "scaling": "strong" if shard else "weak",
           "ms_per_step": ms / steps, "steps": steps, "warmup": warmup,
           "phases_ms_per_step": {k: v[0] / steps for k, v in ph.items()}}
    oz = (False, False, 0)
    if args.propagator == "dense" and prop > 0 and ph.get("ku_mma", (0.0,))[0] > 0:
        # the modular INT8 K U (csrc/ozaki.h): the INT8 launch alone against the INT8 peak
        oz_s = int(os.environ.get("TRAJ_OZAKI_MODULI", "16"))
        mma = ph["ku_mma"][0] / steps
        tops = 2.0 * OZ_NP * oz_s * rows * w.L * w.N / (mma / 1e3) / 1e12
        eq8 = 8.0 * rows * w.L * w.N / (prop / 1e3) / 1e12
        out["roofline_propagate"] = {"bound": "tensor", "achieved": tops, "peak": INT8_PEAK_TOPS, "unit": "TOPS (INT8)",
                                     "frac": tops / INT8_PEAK_TOPS, "kernel_ms": mma, "phase_ms": prop,
                                     "kernel": f"igemm_i8_kernel: the {OZ_NP} x {oz_s} residue products of K U",
                                     "fp64_equiv_tflops": eq8, "fp64_equiv_frac_of_dmma_peak": eq8 / FP64_PEAK_TFLOPS,
                                     "peak_source": INT8_PEAK_SOURCE}
        oz = (True, True, oz_s)
    elif args.propagator == "dense" and prop > 0:
        eq8 = 8.0 * rows * w.L * w.N / (prop / 1e3) / 1e12
        a = 0.75 if P.traj_get_zgemm_algorithm() == "3m" or os.environ.get("TRAJ_PLANAR_KU", "1") != "0" else 1.0
        if os.environ.get("TRAJ_PLANAR_KU", "1") != "0":
            a *= (7 / 8) ** strassen_levels(w, world if shard else 1)   # Strassen levels on each planar product
        out["roofline_propagate"] = {"bound": "tensor", "achieved": eq8 * a, "peak": FP64_PEAK_TFLOPS,
                                     "unit": "TFLOP/s", "frac": eq8 * a / FP64_PEAK_TFLOPS,
                                     "achieved_8mnk_equiv": eq8, "frac_8mnk_equiv": eq8 / FP64_PEAK_TFLOPS,
                                     "flops_counted": "executed DMMA flops (6mnk for 3M, x 7/8 with one Strassen "
                                                      "level)"}
    return out


def run_fp64_path(args, w, tpg, P, steps=3, warmup=2):
    """The step with every contraction on the DMMA (FP64 tensor) kernels, timed the same way."""
    import torch
    old = os.environ.get("TRAJ_OZAKI")
    os.environ["TRAJ_OZAKI"] = "0"
    try:
        tr = open_handle(P, args, w, "traj", 0, 1, tpg)
    finally:
        if old is None:
            os.environ.pop("TRAJ_OZAKI", None)
        else:
            os.environ["TRAJ_OZAKI"] = old
    assert not any(tr.ozaki_info()[:2])
    tr.step(warmup)
    torch.cuda.synchronize()
    tr.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(tr.stream)
    tr.step(steps)
    e1.record(tr.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    ph = tr.phase_times()
    tr.close()
    del tr
    torch.cuda.empty_cache()
    prop = ph["propagate"][0] / steps
    slv = strassen_levels(w, 1, tpg)
    a = 0.75 * (7 / 8) ** slv   # planar 3M (6mnk) x 7/8 per Strassen level: the DMMA flops issued
    eq8 = 8.0 * w.L * w.L * w.N * tpg / (prop / 1e3) / 1e12
    return {"config": "the same workload with TRAJ_OZAKI=0 (planar 3M + Strassen DMMA kernels)",
            "ms_per_step": ms, "value": tpg / (ms / 1e3), "unit": "trajectory-steps/s", "steps": steps,
            "warmup": warmup, "phases_ms_per_step": {k: v[0] / steps for k, v in ph.items() if v[0] > 0},
            "roofline_propagate": {"bound": "tensor", "achieved": eq8 * a, "peak": FP64_PEAK_TFLOPS,
                                   "unit": "TFLOP/s (FP64 DMMA, executed)", "frac": eq8 * a / FP64_PEAK_TFLOPS,
                                   "kernel_ms": prop, "achieved_8mnk_equiv": eq8,
                                   "kernel": f"dgemm_dmma_kernel: planar 3M, {slv} Strassen level(s), split / "
                                             "recombination passes included",
                                   "peak_source": FP64_PEAK_SOURCE}}


def run_e2e(args, w, tpg, mode, rank, world, P):
    """Same metric through the public API from host buffers: the handle is created inside the
    timed region (K built on the device; row-sharded: the NCCL communicator too), the initial
    orbital matrix comes from pinned host memory (traj_set_state; row-sharded: this rank's rows),
    every step ends with a device->host read of the occupations n_i this GPU holds, and the
    config's sampled observables run at its cadence (every w.sample_every steps, as a user's run
    would; SURVEY §8(d) times them separately, `sampled_observables_ms`)."""
    import torch
    shard = mode == "shard"
    rows = w.L // world if shard else w.L
    r0 = rank * rows if shard else 0
    occ = np.arange(0, w.L, 2) if w.Ly == 1 else None
    if occ is None:
        ys, xs = np.divmod(np.arange(w.L), w.Lx)
        occ = np.nonzero((xs + ys) % 2 == 0)[0]
    U0 = torch.zeros((rows, w.N), dtype=torch.complex128).pin_memory()
    sel = (occ >= r0) & (occ < r0 + rows)
    U0[torch.from_numpy(occ[sel] - r0), torch.from_numpy(np.nonzero(sel)[0])] = 1.0
    n_host = torch.empty((tpg, rows), dtype=torch.float64).pin_memory()
    torch.cuda.synchronize()
    if world > 1:
        _dist().barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    t_init = time.perf_counter()
    tr = open_handle(P, args, w, mode, rank, world, tpg, stream=stream)
    init_ms = 1e3 * (time.perf_counter() - t_init)      # traj_init returns after its own stream sync
    for t in range(tpg):
        tr.set_state(t, U0)                       # H2D from pinned host memory
    h2d = tpg * U0.numel() * 16
    d2h = 0
    samples = 0
    for s in range(1, args.steps + 1):
        tr.step(1)
        n_host.copy_(tr.occupations().reshape(tpg, rows), non_blocking=True)   # D2H of the step's result
        d2h += n_host.numel() * 8
        if s % w.sample_every == 0:
            for region in w.regions.values():
                r = tr.mutual_info(*region) if isinstance(region, tuple) else tr.entropy(region)
                d2h += r.size * 8
            samples += 1
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    tr.close()
    ms = max_over_ranks(ms, world)
    return {"value": (1 if shard else world) * tpg * args.steps / (ms / 1e3), "unit": "trajectory-steps/s",
            "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
            "handle_init_ms": init_ms,
            "includes": f"handle init (workspace from torch's caching allocator, K built on the device"
                        f"{', NCCL communicator' if shard and world > 1 else ''}), U0 upload "
                        f"from pinned host{' (this rank' + chr(39) + 's rows)' if shard and world > 1 else ''}, "
                        f"{args.steps} steps with a D2H of n_i after each, the config's observables every "
                        f"{w.sample_every} steps ({samples} sample(s) in this window; their cost alone is "
                        f"sampled_observables_ms)"}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w, tpg = workload(args)
    mode = resolve_mode(args, w, world)
    if mode == "shard":
        tpg = 1
    times, blas = oracle_steps(w, budget_s=args.cpu_budget, max_steps=max(1, args.steps))
    v = len(times) / sum(times)
    unit = "trajectory-steps/s"
    rec = {"metric": "trajectory steps/s (configs[2]: 1d L=16384 projective; metric also quoted at 2d 160x160)",
           "value": v, "unit": unit, "impl": "reference", "n_gpus": world, "steps": len(times), "warmup": 0,
           "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
           "scaling": "strong" if mode == "shard" else "weak",
           "vs_baseline": None, "dtype": "c128 (f64 arithmetic)", "data": "synthetic (Neel start, Philox randoms, seed 0)",
           "config": describe(w, tpg, mode, world, args),
           "note": (f"the oracle (NumPy/SciPy on the host cores) steps one trajectory at a time on rank 0; the "
                    f"{tpg} trajectory(ies) per GPU of the config are independent and cost the same, so the rate "
                    "of one is the config's per-trajectory rate"),
           "cpu_baseline": {"value": v, "unit": unit, "cores": cpu_cores(), "kind": "oracle",
                            "sample": f"{len(times)} oracle step(s) of one {w.name} trajectory (budget "
                                      f"{args.cpu_budget:.0f} s; no warm-up: NumPy has no JIT), {'; '.join(blas)}"},
           "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(rec), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
