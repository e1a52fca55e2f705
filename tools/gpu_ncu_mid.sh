#!/bin/bash
# ncu --set full of one launch of the cluster kernels at the new mid sizes: pair_kernel_f64
# (N = 4096 FP64, K = 2) and pair_kernel K = 4 (N = 8192 FP32), via tools/pair_probe.py.
cd "$(dirname "$0")/.."
O=gpurun_out/ncu_mid; mkdir -p $O
NB_PROBE_PREC=double timeout 300 python tools/pair_probe.py 4096 > $O/probe_f64.log 2>&1 || { cat $O/probe_f64.log; exit 1; }
timeout 300 python tools/pair_probe.py 8192 > $O/probe_f32.log 2>&1 || { cat $O/probe_f32.log; exit 1; }
NB_PROBE_PREC=double timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel_f64 --launch-skip 2 -c 1 \
  -o $O/prof_N4096_f64_pair -f python tools/pair_probe.py 4096 > $O/ncu_f64.log 2>&1; echo "rc=$?" >> $O/ncu_f64.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel --launch-skip 2 -c 1 \
  -o $O/prof_N8192_f32_pair -f python tools/pair_probe.py 8192 > $O/ncu_f32.log 2>&1; echo "rc=$?" >> $O/ncu_f32.log
tail -n 3 $O/*.log; ls -la $O
