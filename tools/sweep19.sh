python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -3
python tools/one_layer.py --reps 20 | tail -2
LOKI_SPLITK=0 python tools/one_layer.py --reps 20 | tail -1
python tools/one_layer.py --reps 20 | tail -1
python tools/one_layer.py --B 32 --H 32 --Hkv 8 --S 32768 --kf 0.125 --df 0.5 --reps 5 | tail -1
LOKI_SPLITK=0 python tools/one_layer.py --B 32 --H 32 --Hkv 8 --S 32768 --kf 0.125 --df 0.5 --reps 5 | tail -1
