set +e
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_ozaki.py -m gpu -x -q -p no:cacheprovider > gpurun_out/t4_oz.log 2>&1; echo "oz rc=$?" >> gpurun_out/t4_oz.log
tail -5 gpurun_out/t4_oz.log
T="timeout 300 python tools/time_step.py --config c3 --warmup 2 --steps 4"
$T 2>&1 | tail -2
TRAJ_OZAKI_MODULI=18 $T 2>&1 | tail -2
timeout 400 python tools/time_step.py --config c5 --warmup 1 --steps 2 2>&1 | tail -2
timeout 2700 python -m pytest tests -m gpu -q -x -p no:cacheprovider --deselect tests/test_gpu_ozaki.py > gpurun_out/t4_all.log 2>&1; echo "all rc=$?" >> gpurun_out/t4_all.log
tail -5 gpurun_out/t4_all.log
