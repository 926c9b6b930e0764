set +e
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s6_gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/s6_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s6_smoke.log 2>&1; echo "smoke rc=$?"
tail -2 gpurun_out/s6_smoke.log
