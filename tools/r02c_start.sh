# Session start: GPU suite, C5 RCM bench, full ncu of the U-mode V-cycle kernels (C5 recipe, 64^3).
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02c_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r02c_gputests.log
timeout 600 python bench.py --ordering rcm --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02c_bench_C5_rcm.json 2> gpurun_out/r02c_bench_C5_rcm.err; echo "bench rc=$?"
timeout 300 python tools/prof_prec.py C5m 1 rcm > gpurun_out/pp.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_vt|k_cg3" -c 4 \
    -o gpurun_out/r02c_full_umode -f python tools/prof_prec.py C5m 1 rcm > gpurun_out/ncu_full_umode.log 2>&1
echo "ncu full rc=$?"
