set +e
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "event or checkpoint" > gpurun_out/s15_test.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/s15_test.log
{ timeout 600 python tools/events_2d_time.py 64 0.3 3; timeout 900 python tools/events_2d_time.py 96 0.3 2; } > gpurun_out/s15_ev2d.txt 2>&1
cat gpurun_out/s15_ev2d.txt
