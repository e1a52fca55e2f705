#!/bin/bash
# pair_probe at several N: stream-K (NB_PAIR=0), pair K=7 (default lib), pair K=6 (variant lib)
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
NS=${NS:-"14208 16384 16576 32768 131072"}
( NB_PAIR=0 timeout 300 python tools/pair_probe.py $NS
  NB_PAIR=1 timeout 300 python tools/pair_probe.py $NS
  NB_PAIR=1 NB_LIB_PATH=tools/variants/lib_pair_k6.so timeout 300 python tools/pair_probe.py 9472 14208 ) > $O/probe.log 2>&1
cat $O/probe.log
