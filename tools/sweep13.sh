python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -6
LOKI_TRACE=1 python tools/one_layer.py --B 32 --H 32 --Hkv 8 --S 32768 --kf 0.125 --df 0.5 --reps 5 | grep -v "CTAs in"
LOKI_TRACE=1 python tools/one_layer.py --B 64 --H 32 --Hkv 8 --S 16384 --kf 0.25 --df 0.25 --reps 5 | grep -v "CTAs in"
python tools/one_layer.py --reps 20
