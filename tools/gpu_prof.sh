cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "from paper_2508_18468_b200 import build; build.build(force=True)" > gpurun_out/r2_build.log 2>&1
T="${R2_TAG:-p}"
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2_${T}_launches_c3.csv python tools/prof_step.py --config c3 --warmup 2 --steps 1 \
  > gpurun_out/r2_${T}_ncu_c3.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2_${T}_ncu_c3.log
