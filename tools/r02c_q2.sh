# Q mode iteration: quick parity, C5 launch list for LP in $QLPS, optional full ncu on C5m.
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_qmode.py -x -q -k "C5s or C5m" > gpurun_out/q_tests.log 2>&1; rc=$?; echo "q tests rc=$rc"; tail -5 gpurun_out/q_tests.log
[ $rc -ne 0 ] && exit 0
export LORPC_QMODE=1
for lp in ${QLPS:-4}; do
  export LORPC_QLP=$lp
  timeout 300 python tools/prof_prec.py C5 2 rcm > gpurun_out/q_pp_$lp.log 2>&1 || { echo "plain run failed lp=$lp"; tail -5 gpurun_out/q_pp_$lp.log; continue; }
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,lts__t_sector_hit_rate.pct --clock-control none \
    -k regex:"k_vq|k_vt" -c 1 --csv --log-file gpurun_out/q_launches_$lp.csv python tools/prof_prec.py C5 1 rcm > gpurun_out/q_ncu_$lp.log 2>&1
  python - <<PY
import csv
rows = [r for r in csv.reader(open("gpurun_out/q_launches_$lp.csv")) if len(r) > 10 and r[0].isdigit()]
for r in rows: print("LP=$lp ${QTAG}", r[4][:24], r[-3], r[-1])
PY
done
if [ -n "$QFULL" ]; then
  export LORPC_QLP=$QFULL
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_vq" -c 1 \
    -o gpurun_out/q_full -f python tools/prof_prec.py C5m 1 rcm > gpurun_out/q_ncu_full.log 2>&1
  echo "ncu full rc=$?"
fi
