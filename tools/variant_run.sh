#!/bin/bash
# usage: tools/variant_run.sh <variant zgemm.cu> ; rebuilds libtraj with it and runs the 3M gemm bench
cp "$1" paper_2508_18468_b200/csrc/zgemm.cu
python paper_2508_18468_b200/build.py --force > /dev/null 2>&1 || { echo build failed; exit 1; }
TRAJ_ZGEMM_3M=1 python tools/gemm_bench.py NN_KU CN_herk_upper NN_trmm
