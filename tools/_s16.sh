LOKI_TUNING=1 LOKI_TRACE=1 LOKI_DEBUG=16 timeout 300 python tools/one_layer.py --B 32 --H 32 --Hkv 8 --S 32768 --kf 0.125 --df 0.5 --reps 5 2>&1 | tail -9
LOKI_TUNING=1 LOKI_TRACE=1 LOKI_DEBUG=16 timeout 300 python tools/one_layer.py --B 64 --H 32 --Hkv 8 --S 16384 --kf 0.25 --df 0.25 --reps 5 2>&1 | tail -9
