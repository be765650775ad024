#!/bin/bash
# One GPU session: build, bench (C5 headline), ncu launch list, ncu full capture of
# the dominant kernel.  Outputs under gpurun_out/ (copy summaries to profiles/).
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 4000 gpurun_out/bench.json
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_vcycle -s 2 -c 1 -o gpurun_out/prof_vcycle_bench \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_cg3 -s 2 -c 1 -o gpurun_out/prof_cg3_bench \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_cg.log 2>&1
echo "ncu cg rc=$?"
