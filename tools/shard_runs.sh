# Row-sharded step timings on one GPU (tools/time_step.py --shards): the NCCL code path on a one-rank
# communicator (--shards 1) and the single-GPU emulation of P shards (every shard's work serialised)
for sh in 1 2 8; do timeout 300 python tools/time_step.py --config c3 --shards $sh --warmup 2 --steps 3; done
TRAJ_SHARD_OZ_CHUNKS=1 timeout 300 python tools/time_step.py --config c3 --shards 8 --warmup 2 --steps 3
TRAJ_OZAKI=0 timeout 300 python tools/time_step.py --config c3 --shards 1 --warmup 2 --steps 3
timeout 300 python tools/time_step.py --config c3 --warmup 2 --steps 3
for sh in 1 2 8; do timeout 600 python tools/time_step.py --config c5 --shards $sh --warmup 1 --steps 2; done
timeout 600 python tools/time_step.py --config c5 --warmup 1 --steps 2
