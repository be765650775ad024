# Deeper-pipelined U sweeps: parity under LORPC_UNST=4, then C5 smoothing-kernel timing per depth.
python -c "import __graft_entry__ as g; g.build()" || exit 1
for n in 3 6; do
LORPC_UNST=$n timeout 900 python -m pytest tests/test_gpu_umode.py -x -q > gpurun_out/unst_tests_$n.log 2>&1; rc=$?; echo "unst=$n tests rc=$rc"; tail -3 gpurun_out/unst_tests_$n.log
[ $rc -ne 0 ] && exit 0
done
for n in ${NSTS:-2 3 4 5 6}; do
  export LORPC_UNST=$n
  timeout 300 python tools/prof_prec.py C5 2 rcm > gpurun_out/unst_pp_$n.log 2>&1 || { echo "plain run failed n=$n"; tail -5 gpurun_out/unst_pp_$n.log; continue; }
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none \
    -k regex:"k_vt_smooth" -c 2 --csv --log-file gpurun_out/unst_launches_$n.csv python tools/prof_prec.py C5 1 rcm > gpurun_out/unst_ncu_$n.log 2>&1
  python - <<PY
import csv
rows = [r for r in csv.reader(open("gpurun_out/unst_launches_$n.csv")) if len(r) > 10 and r[0].isdigit()]
for i in ("0","1"):
    rr = [r for r in rows if r[0]==i]
    print("NST=$n", rr[0][4][:34], " | ".join(f"{r[-3].split('.')[0].split('__')[-1]}={r[-1]}" for r in rr))
PY
done
