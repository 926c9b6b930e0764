set +e
mkdir -p gpurun_out
cat > /tmp/ev1.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2508_18468_b200 as P
tr = P.Trajectories(96, 96, "projective_events", [0.3], seed=0, orthonormalizer="lowrank")
tr.step(1)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
tr.step(1)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(tr.last_clicks(0))
PY
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s16_launches_ev2d.csv python /tmp/ev1.py > gpurun_out/s16_ncu.log 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/s16_launches_ev2d.csv | head -30
