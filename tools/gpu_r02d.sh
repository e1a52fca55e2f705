#!/bin/bash
# Round-2 session d: pair-kernel tests + the GPU suite files touching the step path + C2/C3 bench lines.
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
timeout 2400 python -m pytest -m gpu -q -rs --durations=10 ${PYTEST_ARGS:-tests} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for c in ${CONFIGS:-C2}; do timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
tail -n 5 $O/pytest_gpu.log; tail -n 3 $O/*.err
