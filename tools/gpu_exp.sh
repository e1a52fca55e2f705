cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
NB_VARIANTS=base,f64_mixed timeout 600 python tools/variants.py run C3-f64 C4 > gpurun_out/var_f64.log 2>&1
timeout 300 python tools/diag_bench.py C3-f64 C4 C5 > gpurun_out/diag_base.log 2>&1
NB_DIAG_LEGACY_LIB=tools/variants/lib_f64_mixed.so timeout 300 python tools/diag_bench.py C3-f64 C4 C5 > gpurun_out/diag_mixed.log 2>&1
