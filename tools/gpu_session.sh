#!/bin/bash
# Full GPU session: parity tests, smoke, bench (both arms), ncu launch list + full capture.
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
for c in ${EXTRA_CONFIGS}; do timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
if [ -n "${NCU_CONFIG}" ]; then
  python tools/profile_step.py ${NCU_CONFIG} 3 > $O/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_${NCU_CONFIG}.csv \
      python tools/profile_step.py ${NCU_CONFIG} 3 > $O/ncu_launch.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 1 -c 1 \
      -o $O/prof_${NCU_CONFIG} python tools/profile_step.py ${NCU_CONFIG} 2 > $O/ncu_full.log 2>&1
  echo "ncu rc=$?" >> $O/ncu_full.log
fi
