cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/small_n_bench.py 10 > gpurun_out/small_n.md 2>&1
timeout 300 python bench.py --config C1 > gpurun_out/bench_C1.json 2> gpurun_out/bench_C1.err
