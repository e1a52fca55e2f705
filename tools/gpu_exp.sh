cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
NB_VARIANTS=base,old,base,old timeout 900 python tools/variants.py run C3-f32 C2 C3-f64 > gpurun_out/var_ab.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_a.json 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_b.json 2>&1
