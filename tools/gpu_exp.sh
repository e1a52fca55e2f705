cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python bench.py --config C1 > gpurun_out/bench_C1.json 2> gpurun_out/bench_C1.err
timeout 300 python tools/e2e_breakdown.py C1 > gpurun_out/e2e_C1.txt 2>&1
