set +e
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s14_gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/s14_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s14_smoke.log 2>&1; echo "smoke rc=$?"
tail -1 gpurun_out/s14_smoke.log
timeout 1200 python bench.py > gpurun_out/s14_bench.json 2> gpurun_out/s14_bench.err; echo "bench rc=$?"
tail -c 300 gpurun_out/s14_bench.err
for c in c3 c5; do
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/s14_launches_$c.csv python tools/prof_step.py --config $c --warmup 2 --steps 1 > gpurun_out/s14_ncu_$c.log 2>&1
echo "ncu $c rc=$?"
done
T3="timeout 300 python tools/time_step.py --config c3 --warmup 3 --steps 6"
T5="timeout 400 python tools/time_step.py --config c5 --warmup 2 --steps 3"
{
$T3 2>&1 | tail -1
TRAJ_OZAKI_STRUCT_MIN=64 $T3 2>&1 | tail -1
TRAJ_STRUCT_CHOL=0 $T3 2>&1 | tail -1
$T5 2>&1 | tail -1
TRAJ_STRUCT_CHOL=0 $T5 2>&1 | tail -1
TRAJ_STRUCT_B=1024 $T5 2>&1 | tail -1
} > gpurun_out/s14_exp.txt 2>&1
cat gpurun_out/s14_exp.txt
timeout 600 python bench.py --protocol projective_events --orthonormalizer lowrank --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-observables --secondary none --no-fp64-path 2>&1 | tail -1 | cut -c1-400
