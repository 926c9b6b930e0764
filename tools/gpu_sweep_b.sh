cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "from paper_2508_18468_b200 import build; build.build(force=True)" >/dev/null 2>&1
for b in 512 768 1024; do
  TRAJ_STRUCT_B=$b timeout 600 python bench.py --config c5 --steps 3 --warmup 2 --secondary none --no-cpu-baseline --no-e2e --no-observables > gpurun_out/r2_sweep5_b$b.json 2>/dev/null
done
