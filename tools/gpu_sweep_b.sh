cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "from paper_2508_18468_b200 import build; build.build(force=True)" >/dev/null 2>&1
C="--no-cpu-baseline --no-e2e --no-observables --secondary none --steps 10 --warmup 3"
python bench.py --config c2 $C > gpurun_out/r2_sw_c2_def.json 2>/dev/null
TRAJ_STRASSEN_MIN_N=1024 python bench.py --config c2 $C > gpurun_out/r2_sw_c2_s1.json 2>/dev/null
TRAJ_STRASSEN_MIN_N=1024 TRAJ_STRASSEN_LEVELS=2 python bench.py --config c2 $C > gpurun_out/r2_sw_c2_s2.json 2>/dev/null
python bench.py --config c4 $C > gpurun_out/r2_sw_c4_def.json 2>/dev/null
TRAJ_STRASSEN_LEVELS=2 python bench.py --config c4 $C > gpurun_out/r2_sw_c4_s2.json 2>/dev/null
TRAJ_STRASSEN=0 python bench.py --config c4 $C > gpurun_out/r2_sw_c4_s0.json 2>/dev/null
