#!/bin/bash
# small-N kernel: parity tests, C1 bench line, ncu full capture (excess shared wavefronts)
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest -m gpu -q -x tests/test_gpu_parity.py tests/test_gpu_hostapi.py tests/test_gpu_dropin.py > $O/pt_small.log 2>&1; echo "pytest rc=$?" >> $O/pt_small.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $O/pt_small.log 2>&1; echo "smoke rc=$?" >> $O/pt_small.log
timeout 600 python bench.py --config C1 --no-cpu-baseline --no-traffic > $O/bench_C1.json 2> $O/bench_C1.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:small_simulate_kernel -s 3 -c 1 \
    -o $O/prof_C1_small -f python bench.py --config C1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-traffic > $O/ncu_C1.log 2>&1
tail -3 $O/pt_small.log; tail -1 $O/bench_C1.json | cut -c1-300
