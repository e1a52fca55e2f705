#!/bin/bash
# Round-2 refresh of the judged evidence (outputs in gpurun_out/r02/): smoke, bench lines
# for every BASELINE config (default C3-f32 with the CPU baseline; the reference arm),
# launch lists of the C3-f32 and C2 bench commands, ncu --set full of the shipped
# C3-f32 step kernel and C1 small-N kernel.
cd "$(dirname "$0")/.."
O=gpurun_out/r02; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_C3-f32.json 2> $O/bench_C3-f32.err; echo "bench rc=$?" >> $O/bench_C3-f32.err
for c in C1 C2 C3-f64 C4 C5; do timeout 1500 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
for c in C3-f32 C2; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench_$c.csv \
      python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-traffic > $O/ncu_launch_$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 1 -c 1 \
    -o $O/prof_C3-f32 -f python tools/profile_step.py C3-f32 2 > $O/ncu_full_C3.log 2>&1; echo "ncu rc=$?" >> $O/ncu_full_C3.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:small_simulate_kernel -s 3 -c 1 \
    -o $O/prof_C1_small -f python bench.py --config C1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-traffic > $O/ncu_full_C1.log 2>&1; echo "ncu rc=$?" >> $O/ncu_full_C1.log
ls -la $O; tail -n 2 $O/*.err $O/*.log
