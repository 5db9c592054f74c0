python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -3
python tools/one_layer.py --reps 20 | tail -1
python tools/one_layer.py --S 32768 --reps 10 | tail -1
python tools/one_layer.py --S 16384 --reps 10 | tail -1
LOKI_PIPE_BIG=0 python tools/one_layer.py --S 16384 --reps 10 | tail -1
