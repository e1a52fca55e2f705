cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python tools/cpu_vs_gpu.py > gpurun_out/cpu_vs_gpu.md 2> gpurun_out/cpu_vs_gpu.err
