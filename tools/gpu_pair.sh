#!/bin/bash
# A/B of the cluster split-source kernel (NB_PAIR=0: stream-K + fixup) at C2, plus its parity tests.
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
for p in 0 1; do NB_PAIR=$p NB_VARIANTS=base timeout 600 python tools/variants.py run ${CONFIGS:-C2} > $O/pair_ab_$p.log 2>&1; done
timeout 1200 python -m pytest -m gpu -q -x ${PYTEST_ARGS:-tests/test_gpu_parity.py} > $O/pair_pytest.log 2>&1; echo "pytest rc=$?" >> $O/pair_pytest.log
for c in ${BENCH_CONFIGS:-C2}; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
tail -n 4 $O/pair_ab_*.log $O/pair_pytest.log; cat $O/bench_*.json
