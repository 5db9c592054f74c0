python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -25
LOKI_TRACE=1 python tools/one_layer.py --reps 20
LOKI_PIPE_LAG_X10=12 python tools/one_layer.py --reps 20
LOKI_PIPE_LAG_X10=16 python tools/one_layer.py --reps 20
LOKI_PIPE_LAG_X10=40 python tools/one_layer.py --reps 20
LOKI_TRACE=1 python tools/one_layer.py --S 32768 --reps 10
LOKI_PIPE_LAG_X10=12 python tools/one_layer.py --S 32768 --reps 10
