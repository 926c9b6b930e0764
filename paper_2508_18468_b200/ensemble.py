"""Trajectory-parallel ensembles.

The paper averages its observables over quantum trajectories and over time points
("over quantum trajectories", "over both different trajectories and equally
spaced time points").  Trajectories are independent, so one process per GPU takes a
contiguous block of global trajectory ids (Philox counter word 2) and advances it with
one ``Trajectories`` handle; at each sample time the per-rank sums (sum S, sum S^2,
count) are combined with a single all_reduce.  Failed trajectories (Cholesky breakdown /
bad spectrum) are excluded, never reseeded (SPEC S:558 reading).  No data-path collective
is needed inside a step: this is weak scaling.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def partition(n_traj: int, world: int, rank: int):
    """Contiguous block [start, start+count) of global trajectory ids owned by rank."""
    base, extra = divmod(n_traj, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def moments_to_stats(sums: np.ndarray):
    """(sum, sum of squares, count) along the last axis -> (mean, standard error, count)."""
    s, s2, n = sums[..., 0], sums[..., 1], sums[..., 2]
    with np.errstate(invalid="ignore", divide="ignore"):
        mean = s / n
        var = np.where(n > 1, (s2 - n * mean ** 2) / np.maximum(n - 1, 1), np.nan)
        sem = np.sqrt(np.maximum(var, 0.0) / n)
    return mean, sem, n


def allreduce_sums(sums: np.ndarray, group=None, device=None) -> np.ndarray:
    """Sum the moment arrays over all ranks (one collective for every sample time)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return sums
    t = torch.from_numpy(np.ascontiguousarray(sums, dtype=np.float64))
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.cpu().numpy()


def accumulate(values: np.ndarray, ok: np.ndarray, gamma_index: np.ndarray, n_gamma: int) -> np.ndarray:
    """Per-gamma moments [n_gamma, 3] of the values of the non-failed trajectories."""
    out = np.zeros((n_gamma, 3))
    for v, good, g in zip(values, ok, gamma_index):
        if good and np.isfinite(v):
            out[g] += (v, v * v, 1.0)
    return out


@dataclass
class EnsembleResult:
    times: np.ndarray           # sample steps
    gammas: tuple
    mean: dict                  # observable -> [n_gamma, n_times]
    sem: dict
    count: dict


def _observe(tr, kind: str, region):
    """One sampled observable for every trajectory of the handle.  A spectrum newly found outside
    [-1e-8, 1 + 1e-8] marks that trajectory failed and returns TRAJ_ENUMERIC (traj.h); the call is
    then repeated, giving NaN for the failed one, which ``accumulate`` excludes -- so one bad
    trajectory never aborts the ensemble (nor leaves the other ranks waiting in the all-reduce)."""
    from .binding import TrajError
    for attempt in range(2):
        try:
            return tr.entropy(region) if kind == "entropy" else tr.mutual_info(*region)
        except TrajError as e:
            if e.status != 3 or attempt == 1:
                raise


def run_ensemble(workload, steps: int, sample_every: int, observables: dict, rank: int = 0, world: int = 1,
                 group=None, device=None, max_batch: int | None = None, seed: int | None = None):
    """Advance this rank's block of the workload's trajectories and return ensemble
    statistics (identical on every rank).

    observables: name -> ("entropy", A) or ("mutual_info", (A, B)).
    Trajectory id tau has gamma = workload.gamma_of(tau) (gamma index folded into the id)."""
    import paper_2508_18468_b200 as P
    start, count = partition(workload.n_traj, world, rank)
    ids = np.arange(start, start + count)
    n_gamma = len(workload.gammas)
    gidx = np.array([workload.gammas.index(workload.gamma_of(int(t))) for t in ids], dtype=int)
    times = np.arange(0, steps + 1, sample_every)
    local = {name: np.zeros((len(times), n_gamma, 3)) for name in observables}
    batch = count if max_batch is None else max(1, min(max_batch, count))
    for b0 in range(0, count, batch):
        sub = ids[b0:b0 + batch]
        if sub.size == 0:
            continue
        tr = P.Trajectories(workload.Lx, workload.Ly, workload.protocol, [workload.gamma_of(int(t)) for t in sub],
                            dt=workload.dt, J=workload.J, seed=workload.seed if seed is None else seed,
                            traj_base=int(sub[0]), device=device)
        done = 0
        for k, s in enumerate(times):
            tr.step(int(s - done))
            done = int(s)
            for name, (kind, region) in observables.items():
                vals = _observe(tr, kind, region)
                ok = np.array([not tr.failed(t) for t in range(sub.size)])
                local[name][k] += accumulate(vals, ok, gidx[b0:b0 + batch], n_gamma)
        tr.close()
    mean, sem, cnt = {}, {}, {}
    for name, arr in local.items():
        tot = allreduce_sums(arr, group=group, device=device)
        m, e, n = moments_to_stats(tot)
        mean[name], sem[name], cnt[name] = m.T, e.T, n.T
    return EnsembleResult(times=times, gammas=tuple(workload.gammas), mean=mean, sem=sem, count=cnt)
