set +e
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  --kernel-name regex:"oz_split_cols_kernel|oz_split_rows_kernel|oz_combine_kernel" --launch-count 4 -o gpurun_out/s9_split_full \
  python tools/prof_step.py --config c3 --warmup 2 --steps 1 > gpurun_out/s9_ncu.log 2>&1
echo "ncu rc=$?"
