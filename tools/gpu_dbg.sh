cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "from paper_2508_18468_b200 import build; build.build(force=True)" > gpurun_out/r2_build.log 2>&1
for v in "" "TRAJ_STRUCT_CHOL=0" "TRAJ_STRUCT_CHOL=0 TRAJ_PLANAR_MIN_N=100000" "TRAJ_ZGEMM_3M=0"; do
  timeout 300 python tools/dbg_async.py 512 2.0 3 $v >> gpurun_out/r2_dbg.log 2>&1
done
timeout 300 python tools/dbg_async.py 4096 0.6 2 >> gpurun_out/r2_dbg.log 2>&1
timeout 300 python tools/dbg_async.py 4096 0.6 2 TRAJ_STRUCT_CHOL=0 >> gpurun_out/r2_dbg.log 2>&1
