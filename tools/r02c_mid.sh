# Ring-based mid kernel: parity (thread-mode tests under LORPC_MID_RD=4), then C5 timing per ring depth.
python -c "import __graft_entry__ as g; g.build()" || exit 1
LORPC_MID_RD=4 timeout 900 python -m pytest tests/test_gpu_umode.py tests/test_gpu_parity.py -x -q -k "not wmode" > gpurun_out/mid_tests.log 2>&1; rc=$?; echo "mid tests rc=$rc"; tail -5 gpurun_out/mid_tests.log
[ $rc -ne 0 ] && exit 0
for rd in ${RDS:-0 3 4 6 8}; do
  export LORPC_MID_RD=$rd
  timeout 300 python tools/prof_prec.py C5 2 rcm > gpurun_out/mid_pp_$rd.log 2>&1 || { echo "plain run failed rd=$rd"; tail -5 gpurun_out/mid_pp_$rd.log; continue; }
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct --clock-control none \
    -k regex:"k_vt_mid" -c 1 --csv --log-file gpurun_out/mid_launches_$rd.csv python tools/prof_prec.py C5 1 rcm > gpurun_out/mid_ncu_$rd.log 2>&1
  python - <<PY
import csv
rows = [r for r in csv.reader(open("gpurun_out/mid_launches_$rd.csv")) if len(r) > 10 and r[0].isdigit()]
print("RD=$rd", rows[0][4][:30], " | ".join(f"{r[-3].split('.')[0].split('__')[-1]}={r[-1]}" for r in rows))
PY
done
