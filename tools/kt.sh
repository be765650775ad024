#!/bin/bash
# Quick per-kernel time / DRAM bytes of one C5 preconditioner + operator apply
# under a list of env settings: bash tools/kt.sh "VAR=a VAR2=b" "VAR=c" ...
cfg=${KT_CFG:-C5}
for envs in "$@"; do
  echo "=== $envs"
  env $envs ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:"${KT_K:-k_vt|k_cg3|k_vcycle}" -c ${KT_C:-8} --csv python tools/prof_prec.py $cfg 1 2>/dev/null \
    | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; k=h.index('Kernel Name'); m=h.index('Metric Name'); v=h.index('Metric Value'); u=h.index('Metric Unit'); i=h.index('ID')
cur={}
for r in rows[1:]:
  cur.setdefault((r[i],r[k].split('(')[0]),{})[r[m]]=(r[v],r[u])
for (ii,n),d in cur.items(): print(ii,n[:34].ljust(34),' '.join(f'{a.split(\"__\")[1][:14]}={b[0]}{b[1]}' for a,b in d.items()))
"
done
