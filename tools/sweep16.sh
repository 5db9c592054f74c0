python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -4
LOKI_TRACE=1 LOKI_DEBUG=16 python tools/one_layer.py --reps 10 | grep -v "CTAs in"
LOKI_SPEC=0 python tools/one_layer.py --reps 20 | tail -1
python tools/one_layer.py --reps 20 | tail -1
python tools/one_layer.py --S 32768 --reps 10 | tail -1
LOKI_TRACE=1 python tools/one_layer.py --B 32 --H 32 --Hkv 8 --S 32768 --kf 0.125 --df 0.5 --reps 5 | grep -v "CTAs in"
