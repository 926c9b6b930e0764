set +e
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/s5_bench.json 2> gpurun_out/s5_bench.err; echo "bench rc=$?" >> gpurun_out/s5_bench.err
tail -c 300 gpurun_out/s5_bench.err
for c in c3 c5; do
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/s5_launches_$c.csv python tools/prof_step.py --config $c --warmup 2 --steps 1 > gpurun_out/s5_ncu_$c.log 2>&1
echo "ncu $c rc=$?"
done
timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none \
  --kernel-name regex:igemm_i8_kernel --launch-count 1 -o gpurun_out/s5_ku_full \
  python tools/prof_step.py --config c3 --warmup 2 --steps 1 > gpurun_out/s5_ncu_full.log 2>&1
echo "ncu full rc=$?"
T5="timeout 400 python tools/time_step.py --config c5 --warmup 1 --steps 2"
TRAJ_STRUCT_B=512 $T5 2>&1 | tail -1
TRAJ_STRUCT_B=1024 $T5 2>&1 | tail -1
TRAJ_STRUCT_B=4096 $T5 2>&1 | tail -1
TRAJ_OZAKI_PROJ_MIN=64 timeout 300 python tools/time_step.py --config c3 --warmup 2 --steps 4 2>&1 | tail -1
