cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
NB_VARIANTS=base,unscaled timeout 600 python tools/variants.py run C3-f32 C2 > gpurun_out/var_scaled.log 2>&1
timeout 600 python tools/small_n_bench.py 10 1024,2048,4096 > gpurun_out/small_n.md 2>&1
