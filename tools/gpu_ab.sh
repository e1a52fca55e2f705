#!/bin/bash
# A/B of kernel variants (tools/variants.py) on the GPU: NB_VARIANTS selects,
# CONFIGS the BASELINE configs.  Output: gpurun_out/variants_ab.log + variants.json
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
NB_VARIANTS=${NB_VARIANTS} timeout 1500 python tools/variants.py run ${CONFIGS:-C2 C3-f32 C3-f64} > $O/variants_ab.log 2>&1; echo "rc=$?" >> $O/variants_ab.log
tail -n 30 $O/variants_ab.log
