set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_s3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_s3.log
timeout 900 python bench.py > gpurun_out/bench_s3.json 2> gpurun_out/bench_s3.err; echo "bench rc=$?"
tail -3 gpurun_out/gputest_s3.log
