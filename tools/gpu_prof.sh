#!/bin/bash
# ncu pass on the current build: launch list of one C5 bench step and full
# captures of the preconditioner kernels and the operator (one apply each).
# Usage (on the GPU box): bash tools/gpu_prof.sh [tag]
tag=${1:-cur}
python -c "import __graft_entry__ as g; g.build()" || exit 1
python tools/prof_prec.py C5 2 > gpurun_out/prof_prec_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches_$tag.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches_$tag.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_vt|k_cg3|k_gmg|k_coarse" -s 0 -c 12 \
    -o gpurun_out/prof_$tag -f python tools/prof_prec.py C5 2 > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu full rc=$?"
