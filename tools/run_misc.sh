cd $GRAFT_REPO_ROOT
python tools/variants.py run C2 C3-f32 > gpurun_out/variants.log 2>&1
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
timeout 1200 python bench.py --config C5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
