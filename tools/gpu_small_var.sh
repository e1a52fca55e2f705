#!/bin/bash
# small_n_bench for each variant library in VARS (NS: sizes)
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
: > $O/small_var.log
for v in ${VARS:-base}; do echo "== $v" >> $O/small_var.log
  NB_LIB_PATH=tools/variants/lib_$v.so timeout 600 python tools/small_n_bench.py 10 ${NS:-1024,2048,4096} >> $O/small_var.log 2>&1; done
cat $O/small_var.log
