cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
NB_VARIANTS=base,k4_p4_3of8,k4_p4_2of8 timeout 600 python tools/variants.py run C2 C3-f32 > gpurun_out/var_k4.log 2>&1
