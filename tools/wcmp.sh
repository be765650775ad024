# dev probe: W-mode variants vs thread mode on the C5 recipe at 64^3
python tools/wcheck.py 2>&1 | tail -5
export LORPC_VERBOSE=1
for lp in 16 32; do LORPC_WLP=$lp python tools/wprof.py ${1:-64} 5 2>&1 | tail -2; done
LORPC_WMODE=0 python tools/wprof.py ${1:-64} 5 2>&1 | tail -1
