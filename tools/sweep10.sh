python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -5
LOKI_TRACE=1 LOKI_DEBUG=16 python tools/one_layer.py --reps 5
python tools/one_layer.py --reps 20
LOKI_PIPE_LAG_X10=60 python tools/one_layer.py --reps 20
LOKI_PIPE_LAG_X10=100 python tools/one_layer.py --reps 20
LOKI_TRACE=1 LOKI_DEBUG=16 python tools/one_layer.py --S 32768 --reps 3
python tools/one_layer.py --S 32768 --reps 10
