LOKI_TRACE=1 python tools/one_layer.py --B 32 --H 32 --Hkv 8 --S 32768 --kf 0.125 --df 0.5 --reps 5 | grep -v "CTAs in"
LOKI_PIPE_LAG_X10=100 python tools/one_layer.py --B 32 --H 32 --Hkv 8 --S 32768 --kf 0.125 --df 0.5 --reps 5 | grep -v "CTAs in"
LOKI_TRACE=1 python tools/one_layer.py --reps 10 | grep -v "CTAs in"
