#!/bin/bash
# One GPU session: build check, parity tests, quick perf.  Output in gpurun_out/.
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/clocks_round.csv &
CP=$!
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/perf_quick.py > gpurun_out/perf_quick.log 2>&1; echo "perf rc=$?" >> gpurun_out/perf_quick.log
kill $CP
