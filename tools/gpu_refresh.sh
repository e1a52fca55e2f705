#!/bin/bash
# Round-end refresh of the judged evidence: tests, smoke, bench lines (both arms),
# launch list of the bench command, ncu --set full of the C3-f32 step kernel.
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
for c in C2 C3-f64; do timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 1 -c 1 \
    -o $O/prof_C3-f32 python tools/profile_step.py C3-f32 2 > $O/ncu_full.log 2>&1; echo "ncu rc=$?" >> $O/ncu_full.log
ncu -i $O/prof_C3-f32.ncu-rep --page details --csv > $O/ncu_details_C3-f32.csv 2>/dev/null
