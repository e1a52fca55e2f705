#!/bin/bash
# C1 end-to-end: host phases (trace build), cProfile of the Python side, the C1 bench line, host-API tests.
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest -m gpu -q -x ${PYTEST_ARGS:-tests/test_gpu_hostapi.py tests/test_gpu_dropin.py} > $O/pytest_c1.log 2>&1; echo "pytest rc=$?" >> $O/pytest_c1.log
NB_LIB_PATH=tools/variants/lib_trace.so timeout 300 python tools/host_trace.py C1 300 > $O/host_trace.txt 2>&1
timeout 300 python tools/py_profile.py C1 2000 > $O/py_profile.txt 2>&1
timeout 600 python bench.py --config C1 --no-cpu-baseline > $O/bench_C1.json 2> $O/bench_C1.err
tail -4 $O/pytest_c1.log; cat $O/host_trace.txt; head -25 $O/py_profile.txt; tail -2 $O/bench_C1.err
