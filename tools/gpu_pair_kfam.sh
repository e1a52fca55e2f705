#!/bin/bash
# pair_kernel with K = 2..7 targets per lane (NB_PAIR_K variant libraries) at the N each
# K's 74 clusters cover, against the shipped selection (stream-K / small / persistent).
cd "$(dirname "$0")/.."
O=gpurun_out/pair_kfam; mkdir -p $O
python tools/pair_probe.py 4096 4736 6144 7104 8192 9000 9472 10000 11000 11840 13000 14208 > $O/auto.log 2>&1
NB_PAIR=0 python tools/pair_probe.py 4096 4736 6144 7104 8192 9472 > $O/streamk.log 2>&1
for k in 2 3 4 5 6; do
  case $k in 2) NS="3800 4096 4400 4736";; 3) NS="5600 6144 6600 7104";; 4) NS="7600 8192 9000 9472";; 5) NS="10000 11000 11840";; 6) NS="12000 13000 13600 14208";; esac
  NB_LIB_PATH=$PWD/tools/variants/lib_pair_k$k.so NB_PAIR=1 python tools/pair_probe.py $NS > $O/pair_k$k.log 2>&1
done
tail -n 20 $O/*.log
