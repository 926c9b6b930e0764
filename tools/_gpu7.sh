set +e
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ozaki.py -m gpu -x -q -s -k "tiers" > gpurun_out/s7_test.log 2>&1; echo "pytest rc=$?"
grep -a "delta\|passed\|failed\|Error\|assert" gpurun_out/s7_test.log | tail -30
