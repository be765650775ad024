# Q mode: parity tests, then C5 timing (ncu launch list with DRAM bytes) for LP = 4, 2, 8.
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_qmode.py -x -q > gpurun_out/q_tests.log 2>&1; rc=$?; echo "q tests rc=$rc"; tail -15 gpurun_out/q_tests.log
[ $rc -ne 0 ] && exit 0
for lp in ${QLPS:-4 2 8}; do
  export LORPC_QMODE=1 LORPC_QLP=$lp LORPC_VERBOSE=1
  timeout 300 python tools/prof_prec.py C5 2 rcm > gpurun_out/q_pp_$lp.log 2>&1 || { echo "plain run failed lp=$lp"; tail -5 gpurun_out/q_pp_$lp.log; continue; }
  grep qrec gpurun_out/q_pp_$lp.log
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none \
    -k regex:"k_vq|k_vt" -c 2 --csv --log-file gpurun_out/q_launches_$lp.csv python tools/prof_prec.py C5 2 rcm > gpurun_out/q_ncu_$lp.log 2>&1
  python - <<PY
import csv
rows = [r for r in csv.reader(open("gpurun_out/q_launches_$lp.csv")) if len(r) > 10 and r[0].isdigit()]
for r in rows: print("LP=$lp", r[0], r[4][:40], r[-3], r[-2], r[-1])
PY
done
