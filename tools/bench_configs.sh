#!/bin/bash
# One bench line per BASELINE config at N = 1 (c3 and c5 in dense, banded and banded + low-rank
# forms), appended to gpurun_out/bench_configs.jsonl.  Usage (on the GPU box): bash tools/bench_configs.sh
out=gpurun_out/${BENCH_CONFIGS_OUT:-bench_configs.jsonl}
: > $out
common="--no-cpu-baseline --no-e2e --no-observables --secondary none --no-fp64-path"
python bench.py --config c1 --steps 200 --warmup 10 $common >> $out 2>/dev/null
for c in c2 c4; do
  python bench.py --config $c --steps 10 --warmup 3 $common >> $out 2>/dev/null
done
python bench.py --config c4 --propagator banded --steps 10 --warmup 3 $common >> $out 2>/dev/null
python bench.py --config c2 --propagator banded --steps 10 --warmup 3 $common >> $out 2>/dev/null
python bench.py --config c5 --steps 2 --warmup 2 $common >> $out 2>/dev/null
python bench.py --config c5 --propagator banded --steps 3 --warmup 2 $common >> $out 2>/dev/null
python bench.py --config c5 --propagator banded --orthonormalizer lowrank --steps 3 --warmup 2 $common >> $out 2>/dev/null
python bench.py --orthonormalizer lowrank --steps 5 --warmup 3 $common >> $out 2>/dev/null
python bench.py --propagator banded --steps 5 --warmup 3 $common >> $out 2>/dev/null
python bench.py --propagator banded --orthonormalizer lowrank --steps 10 --warmup 3 $common >> $out 2>/dev/null
python bench.py --protocol homodyne --steps 5 --warmup 3 $common >> $out 2>/dev/null
python bench.py --protocol homodyne_rk4 --steps 5 --warmup 3 $common >> $out 2>/dev/null
python bench.py --protocol projective_events --steps 3 --warmup 2 $common >> $out 2>/dev/null
python bench.py --protocol projective_events --orthonormalizer lowrank --steps 3 --warmup 2 $common >> $out 2>/dev/null
# the DMMA contractions instead of the modular INT8 products (A/B of the round-2 engine)
TRAJ_OZAKI=0 python bench.py --steps 5 --warmup 3 $common >> $out 2>/dev/null
TRAJ_OZAKI=0 python bench.py --config c5 --steps 2 --warmup 2 $common >> $out 2>/dev/null
