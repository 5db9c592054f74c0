python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -3
LOKI_TRACE=1 python tools/one_layer.py --reps 20 | grep -v "CTAs in"
python tools/one_layer.py --S 32768 --reps 10 | tail -1
