# ncu evidence for the c3 propagate phase (round 2): launch list with DRAM bytes of one step, and a
# --set full capture of the batch-21 Strassen K U launch.  Writes gpurun_out/r2_<tag>_*
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "from paper_2508_18468_b200 import build; build.build(force=True)" > gpurun_out/r2_build.log 2>&1
T="${R2_TAG:-n}"
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/r2_${T}_launches_dram_c3.csv \
  python tools/prof_step.py --config c3 --warmup 2 --steps 1 > gpurun_out/r2_${T}_ncu1.log 2>&1
echo "ncu1 rc=$?" >> gpurun_out/r2_${T}_ncu1.log
timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none \
  --kernel-name regex:dgemm_dmma_kernel --launch-count 1 -o gpurun_out/r2_${T}_ku_full \
  python tools/prof_step.py --config c3 --warmup 2 --steps 1 > gpurun_out/r2_${T}_ncu2.log 2>&1
echo "ncu2 rc=$?" >> gpurun_out/r2_${T}_ncu2.log
