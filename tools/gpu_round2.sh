# round-2 GPU session script (run under gpurun from the repo root); writes gpurun_out/r2_<tag>_*
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "from paper_2508_18468_b200 import build; build.build(force=True)" > gpurun_out/r2_build.log 2>&1
T="${R2_TAG:-x}"
if [ -n "${R2_FIRST:-}" ]; then
  timeout 1200 python -m pytest -q -x $R2_FIRST > gpurun_out/r2_${T}_first.log 2>&1
  echo "first rc=$?" >> gpurun_out/r2_${T}_first.log
fi
if [ -z "${R2_SKIP_ALL:-}" ]; then
  timeout 2700 python -m pytest tests -m gpu -q ${R2_PYTEST_ARGS:-} > gpurun_out/r2_${T}_tall.log 2>&1
  echo "tall rc=$?" >> gpurun_out/r2_${T}_tall.log
fi
timeout 900 python bench.py ${R2_BENCH_ARGS:-} > gpurun_out/r2_${T}_bench.json 2> gpurun_out/r2_${T}_bench.err
echo "bench rc=$?" >> gpurun_out/r2_${T}_bench.err
