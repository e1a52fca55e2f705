#!/bin/bash
# ncu --set full of one pair_kernel launch at C2 (cluster split-source kernel).
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
timeout 600 python tools/profile_step.py C2 3 > $O/pstep.log 2>&1 || { cat $O/pstep.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel --launch-skip 1 -c 1 \
  -o $O/prof_C2_pair -f python tools/profile_step.py C2 3 > $O/ncu_pair.log 2>&1
tail -3 $O/ncu_pair.log
