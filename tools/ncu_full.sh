#!/bin/bash
# Full ncu capture (source-level) of the V-cycle kernels on the 64^3 C5 recipe.
# Usage: bash tools/ncu_full.sh tag [kernel-regex]
tag=${1:-cur}; kre=${2:-k_vt}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$kre" -c ${NCU_C:-3} \
    -o gpurun_out/full_$tag -f python tools/prof_prec.py C5m 1 > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu full rc=$?"
