#!/bin/bash
# Small-N kernel's tagged position exchange (NB_SMALL_TAGGED=1, default) vs a grid
# barrier per step (=0): parity/host-API suites with it on, C1 bench lines both ways,
# small-N sweep both ways.  Output: gpurun_out/c1_tagged/
cd "$(dirname "$0")/.."
O=gpurun_out/c1_tagged; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hostapi.py tests/test_gpu_dropin.py -m gpu -x -q --timeout 300 > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for t in 1 0; do
  NB_SMALL_TAGGED=$t timeout 300 python bench.py --config C1 --no-cpu-baseline --no-traffic > $O/bench_C1_tagged$t.json 2> $O/bench_C1_tagged$t.err; echo "rc=$?" >> $O/bench_C1_tagged$t.err
  NB_SMALL_TAGGED=$t timeout 600 python tools/small_n_bench.py > $O/small_n_tagged$t.md 2>&1
done
tail -n 4 $O/pytest.log; for t in 1 0; do python - <<P
import json
d=json.loads(open("$O/bench_C1_tagged$t.json").read().strip().splitlines()[-1])
print("tagged=$t value", d["value"], "e2e", d["e2e"]["value"], "ms_per_step", d["ms_per_step"])
P
done
