set +e
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ozaki.py -m gpu -x -q -p no:cacheprovider -k "structured or modular or projective or golden" > gpurun_out/t3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t3.log
T="timeout 300 python tools/time_step.py --config c3 --warmup 2 --steps 4"
$T
TRAJ_STRUCT_BATCHED=0 $T
TRAJ_STRUCT_B=64 $T
TRAJ_STRUCT_B=256 $T
TRAJ_STRUCT_B=512 $T
T5="timeout 400 python tools/time_step.py --config c5 --warmup 1 --steps 2"
$T5
