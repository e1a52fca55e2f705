cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
NB_VARIANTS=base,t512_k2,t512_k2_p3,t512_k2_u8,t512_k2_smem timeout 900 python tools/variants.py run C3-f32 C2 > gpurun_out/var_occ.log 2>&1
