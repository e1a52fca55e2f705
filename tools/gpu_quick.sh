#!/bin/bash
# Quick GPU check: selected tests (PYTEST_ARGS), host-overhead breakdown, bench lines (CONFIGS).
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest -m gpu -q -rs ${PYTEST_ARGS:-tests} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python tools/host_overhead.py C1 > $O/host_overhead_C1.txt 2>&1
for c in ${CONFIGS:-C1}; do timeout 900 python bench.py --config $c --no-cpu-baseline ${BENCH_ARGS} > $O/bench_$c.json 2> $O/bench_$c.err; done
tail -n 3 $O/*.log $O/*.err
