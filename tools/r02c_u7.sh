# U sweeps specialised for columns of at most 7 pairs: parity, then C5 timing vs the 13-pair kernels.
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_umode.py "tests/test_gpu_large.py::test_c5_recipe_32cubed_multi_tile" tests/test_gpu_parity.py -x -q -k "not wmode" > gpurun_out/u7_tests.log 2>&1; rc=$?; echo "u7 tests rc=$rc"; tail -3 gpurun_out/u7_tests.log
[ $rc -ne 0 ] && exit 0
for v in 7 13; do
  if [ $v = 13 ]; then export LORPC_UMP13=1; fi
  timeout 300 python tools/prof_prec.py C5 2 rcm > gpurun_out/u7_pp_$v.log 2>&1 || { echo "plain run failed v=$v"; tail -5 gpurun_out/u7_pp_$v.log; continue; }
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none \
    -k regex:"k_vt_" -c 3 --csv --log-file gpurun_out/u7_launches_$v.csv python tools/prof_prec.py C5 1 rcm > gpurun_out/u7_ncu_$v.log 2>&1
  python - <<PY
import csv
rows = [r for r in csv.reader(open("gpurun_out/u7_launches_$v.csv")) if len(r) > 10 and r[0].isdigit()]
for i in sorted(set(r[0] for r in rows)):
    rr = [r for r in rows if r[0]==i]
    print("MPT=$v", rr[0][4][:36], " | ".join(f"{r[-3].split('.')[0].split('__')[-1]}={r[-1]}" for r in rr))
PY
done
