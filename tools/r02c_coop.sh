# Cooperative-row mid kernel: parity (U-mode tests + 32^3 multi-tile), then C5 timing per NBUF.
python -c "import __graft_entry__ as g; g.build()" || exit 1
export LORPC_MID_COOP=1
timeout 600 python -m pytest tests/test_gpu_umode.py "tests/test_gpu_large.py::test_c5_recipe_32cubed_multi_tile" -x -q > gpurun_out/coop_tests.log 2>&1; rc=$?; echo "coop tests rc=$rc"; tail -5 gpurun_out/coop_tests.log
[ $rc -ne 0 ] && exit 0
for nb in ${NBS:-1 2 3}; do
  export LORPC_MID_NBUF=$nb
  timeout 300 python tools/prof_prec.py C5 2 rcm > gpurun_out/coop_pp_$nb.log 2>&1 || { echo "plain run failed nb=$nb"; tail -5 gpurun_out/coop_pp_$nb.log; continue; }
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct --clock-control none \
    -k regex:"k_vt_" -c 4 --csv --log-file gpurun_out/coop_launches_$nb.csv python tools/prof_prec.py C5 1 rcm > gpurun_out/coop_ncu_$nb.log 2>&1
  python - <<PY
import csv
rows = [r for r in csv.reader(open("gpurun_out/coop_launches_$nb.csv")) if len(r) > 10 and r[0].isdigit()]
for i in sorted(set(r[0] for r in rows)):
    rr = [r for r in rows if r[0]==i]
    print("NBUF=$nb", rr[0][4][:34], " | ".join(f"{r[-3].split('.')[0].split('__')[-1]}={r[-1]}" for r in rr))
PY
done
