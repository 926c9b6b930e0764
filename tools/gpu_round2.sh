cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt 2>&1
python -c "from paper_2508_18468_b200 import build; build.build(force=True)" > gpurun_out/r2_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_golden_full.py tests/test_gpu_api.py -q -x --deselect "tests/test_gpu_golden_full.py::test_full_size_matches_oracle_golden[c5]" > gpurun_out/r2_t1.log 2>&1
echo "t1 rc=$?" >> gpurun_out/r2_t1.log
timeout 2400 python -m pytest tests -m gpu -q --deselect "tests/test_gpu_golden_full.py::test_full_size_matches_oracle_golden[c5]" > gpurun_out/r2_tall.log 2>&1
echo "tall rc=$?" >> gpurun_out/r2_tall.log
timeout 900 python bench.py > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err
echo "bench rc=$?" >> gpurun_out/r2_bench1.err
