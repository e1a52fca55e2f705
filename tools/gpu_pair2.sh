#!/bin/bash
# pair kernel: tests, probe, ncu full capture at C2
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest -m gpu -q -x tests/test_gpu_pair.py tests/test_gpu_fixup.py > $O/pt_pair.log 2>&1; echo "pytest rc=$?" >> $O/pt_pair.log
NB_PAIR=1 timeout 300 python tools/pair_probe.py 16576 --j 4096,16576 > $O/probe_pair.log 2>&1
bash tools/gpu_ncu_pair.sh > /dev/null 2>&1
tail -2 $O/pt_pair.log; cat $O/probe_pair.log
