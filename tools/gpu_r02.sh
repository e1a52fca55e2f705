#!/bin/bash
# Round-2 GPU session: every GPU test (with durations), smoke, bench lines (both
# arms, default + C1/C2/C3-f64), ncu --set full of the shipped FP64 step kernel
# (C3-f64) and of the FP32 step kernel at C2.  Output in gpurun_out/.
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=25 ${PYTEST_ARGS} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?" >> $O/bench_ref.err
for c in ${EXTRA_CONFIGS:-C1 C2 C3-f64}; do timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
for c in ${NCU_CONFIGS:-C3-f64 C2}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 1 -c 1 \
      -o $O/prof_$c python tools/profile_step.py $c 3 > $O/ncu_full_$c.log 2>&1; echo "ncu rc=$?" >> $O/ncu_full_$c.log
  ncu -i $O/prof_$c.ncu-rep --page raw --csv > $O/ncu_raw_$c.csv 2>/dev/null
  ncu -i $O/prof_$c.ncu-rep --page details --csv > $O/ncu_details_$c.csv 2>/dev/null
done
tail -n 3 $O/*.log $O/*.err
