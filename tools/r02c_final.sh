# Round-2 final measurement pass on one B200: GPU suite, bench lines (C5 headline with RCM and with MDF,
# C4 = three SIPG solves, C3, C2), launch list of one C5 iteration, ncu full of the C5-recipe kernels at 64^3.
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02c_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r02c_gputests.log
python bench.py --steps 5 --warmup 3 > gpurun_out/r02c_bench_C5.json 2> gpurun_out/r02c_bench_C5.err; echo "C5 rc=$?"
python bench.py --ordering mdf --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02c_bench_C5_mdf.json 2> gpurun_out/r02c_bench_C5_mdf.err; echo "C5 mdf rc=$?"
for c in C4 C3 C2; do
  python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02c_bench_$c.json 2> gpurun_out/r02c_bench_$c.err
  echo "$c rc=$?"
done
python tools/prof_prec.py C5 2 rcm > gpurun_out/prof_prec_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_vt|k_cg3|k_pre|k_dot|k_update|k_prolong|k_restrict|k_jacobi|k_residual|k_coarsest" \
    -c 40 --csv --log-file gpurun_out/r02c_launches_C5.csv python tools/prof_prec.py C5 2 rcm > gpurun_out/ncu_l.log 2>&1
echo "launch list rc=$?"
python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02c_launches_bench_C5.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_lb.log 2>&1
echo "bench launch list rc=$?"
python tools/prof_prec.py C5m 2 rcm > gpurun_out/prof_prec_plain_m.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_vt|k_cg3" -s 0 -c 4 \
    -o gpurun_out/r02c_prof_C5m -f python tools/prof_prec.py C5m 1 rcm > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
