LOKI_TRACE=1 python tools/one_layer.py --reps 20 | grep -v "CTAs in"
LOKI_LEAD_LPR=0 python tools/one_layer.py --reps 20 | tail -1
