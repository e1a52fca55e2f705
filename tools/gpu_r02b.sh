#!/bin/bash
# Round-2 session b: GPU tests (full, with printed parity numbers for the large
# and drop-in files), bench lines (default, C1, C2, C3-f64, C5), in-kernel vs
# kernel fixup A/B, per-rank shard compute for C3-f32/C4/C5.
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=15 ${PYTEST_ARGS} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python -m pytest tests/test_gpu_large.py tests/test_gpu_dropin.py tests/test_gpu_ladder.py -m gpu -q -rP -k "not c4_full" > $O/pytest_printed.log 2>&1; echo "rc=$?" >> $O/pytest_printed.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
for c in C1 C2 C3-f64 C5; do timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
for c in C2 C3-f32; do NB_FIXUP_KERNEL=1 timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e --no-traffic > $O/bench_fixk_$c.json 2> $O/bench_fixk_$c.err; done
timeout 900 python tools/shard_scaling.py C3-f32 C4 C5 > $O/shard_scaling.md 2> $O/shard_scaling.err
tail -n 3 $O/*.log $O/*.err
