# U-record kernels: parity, then C5 bench with RCM (U mode) and a launch list.
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_umode.py tests/test_gpu_large.py::test_c5_recipe_32cubed_multi_tile -x -q > gpurun_out/umode_tests.log 2>&1
echo "umode tests rc=$?"; tail -3 gpurun_out/umode_tests.log
timeout 600 python bench.py --ordering rcm --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/umode_bench_C5.json 2> gpurun_out/umode_bench_C5.err
echo "bench rc=$?"
timeout 300 python tools/prof_prec.py C5 2 rcm > gpurun_out/umode_prof_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_vt|k_cg3" -c 8 --csv --log-file gpurun_out/umode_launches_C5.csv python tools/prof_prec.py C5 2 rcm > gpurun_out/umode_ncu_l.log 2>&1
echo "launch list rc=$?"
