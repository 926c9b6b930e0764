set +e
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s19_gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/s19_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s19_smoke.log 2>&1; echo "smoke rc=$?"
tail -1 gpurun_out/s19_smoke.log
timeout 1200 python bench.py > gpurun_out/s19_bench.json 2> gpurun_out/s19_bench.err; echo "bench rc=$?"
tail -c 300 gpurun_out/s19_bench.err
for c in c3 c5; do
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/s19_launches_$c.csv python tools/prof_step.py --config $c --warmup 2 --steps 1 > gpurun_out/s19_ncu_$c.log 2>&1
echo "ncu $c rc=$?"
done
