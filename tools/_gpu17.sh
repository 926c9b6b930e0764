set +e
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "event or checkpoint" --durations=5 > gpurun_out/s17_test.log 2>&1; echo "pytest rc=$?"
tail -12 gpurun_out/s17_test.log
{ timeout 600 python tools/events_2d_time.py 64 0.3 3; timeout 900 python tools/events_2d_time.py 96 0.3 2; } > gpurun_out/s17_ev2d.txt 2>&1
cat gpurun_out/s17_ev2d.txt
timeout 600 python bench.py --protocol projective_events --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-observables --secondary none --no-fp64-path 2>&1 | tail -1 | cut -c1-330
