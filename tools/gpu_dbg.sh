cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "from paper_2508_18468_b200 import build; build.build(force=True)" > gpurun_out/r2_build.log 2>&1
for v in "" "TRAJ_STRUCT_CHOL=0"; do
  timeout 300 python tools/dbg_shard2.py 256 2 3 $v >> gpurun_out/r2_dbg.log 2>&1
done
