# dev probe: C5 bench with / without the R_0 overlap on the aux stream
for o in 0 1; do LORPC_OVERLAP=$o python bench.py --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('overlap', $o, d['value'], d['roofline']['launch_ms'], d['ms_per_step'], d['roofline_operator']['launch_ms'])"; done
