set +e
mkdir -p gpurun_out
T3="timeout 300 python tools/time_step.py --config c3 --warmup 3 --steps 6"
T5="timeout 400 python tools/time_step.py --config c5 --warmup 1 --steps 3"
$T3 2>&1 | tail -1
TRAJ_OZAKI_PRESPLIT=0 $T3 2>&1 | tail -1
$T5 2>&1 | tail -1
TRAJ_OZAKI_PRESPLIT=0 $T5 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_golden_full.py -m gpu -x -q > gpurun_out/s11_test.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/s11_test.log
