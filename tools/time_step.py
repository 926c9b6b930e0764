"""Device time per step and per phase of a config (CUDA events on the handle's stream), for A/B runs of
environment switches: python tools/time_step.py --config c5 --warmup 1 --steps 2"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
import paper_2508_18468_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--shards", type=int, default=0,
                help="row-sharded handle: 1 = the NCCL code path on a one-rank communicator, P > 1 = the "
                     "single-GPU emulation of P shards (every shard's work serialised on this GPU)")
a = ap.parse_args()
w = workloads.CONFIGS[a.config]()
kw = {}
if a.shards == 1:
    kw = dict(shard_size=1, shard_rank=0, nccl_id=P.traj_nccl_unique_id())
elif a.shards > 1:
    kw = dict(shard_size=a.shards)
tr = P.Trajectories(w.Lx, w.Ly, w.protocol, [w.gamma_of(0)], dt=w.dt, seed=w.seed, **kw)
tr.step(a.warmup)
torch.cuda.synchronize()
tr.profile(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(tr.stream)
tr.step(a.steps)
e1.record(tr.stream)
torch.cuda.synchronize()
ph = tr.phase_times()
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("TRAJ_"))
try:
    gd = " gram_dev=" + ",".join(f"{v:.2e}" for v in tr.gram_deviation())
except Exception:
    gd = ""
print(f"{a.config}{f' shards={a.shards}' if a.shards else ''}{gd} oz={tr.ozaki_info()} [{env}] {e0.elapsed_time(e1) / a.steps:.1f} ms/step  " +
      " ".join(f"{k}={v[0] / a.steps:.1f}" for k, v in ph.items() if v[0] > 0), flush=True)
