#!/bin/bash
# pair_probe (NB_PAIR=1) at N (default 16576) for each variant library in VARS
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
: > $O/probe_var.log
for v in ${VARS:-base}; do echo "== $v" >> $O/probe_var.log
  NB_PAIR=1 NB_LIB_PATH=tools/variants/lib_$v.so timeout 300 python tools/pair_probe.py ${NS:-16576} --j 4096,${NS:-16576} >> $O/probe_var.log 2>&1; done
cat $O/probe_var.log
