# smem-staged mid kernel: parity (U-mode + T-mode tests), then C5 timing (RCM and MDF).
python -c "import __graft_entry__ as g; g.build()" || exit 1
export LORPC_MID_SMEM=1
timeout 900 python -m pytest tests/test_gpu_umode.py tests/test_gpu_parity.py "tests/test_gpu_large.py::test_c5_recipe_32cubed_multi_tile" -x -q -k "not wmode" > gpurun_out/mids_tests.log 2>&1; rc=$?; echo "mids tests rc=$rc"; tail -5 gpurun_out/mids_tests.log
[ $rc -ne 0 ] && exit 0
for ord in rcm mdf; do
  timeout 300 python tools/prof_prec.py C5 2 $ord > gpurun_out/mids_pp_$ord.log 2>&1 || { echo "plain run failed $ord"; tail -5 gpurun_out/mids_pp_$ord.log; continue; }
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct --clock-control none \
    -k regex:"k_vt_" -c 3 --csv --log-file gpurun_out/mids_launches_$ord.csv python tools/prof_prec.py C5 1 $ord > gpurun_out/mids_ncu_$ord.log 2>&1
  python - <<PY
import csv
rows = [r for r in csv.reader(open("gpurun_out/mids_launches_$ord.csv")) if len(r) > 10 and r[0].isdigit()]
for i in sorted(set(r[0] for r in rows)):
    rr = [r for r in rows if r[0]==i]
    print("$ord", rr[0][4][:34], " | ".join(f"{r[-3].split('.')[0].split('__')[-1]}={r[-1]}" for r in rr))
PY
done
