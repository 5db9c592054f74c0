python -m pytest tests -m gpu -x -q 2>&1 | tail -5
LOKI_TRACE=1 python tools/one_layer.py --reps 20
LOKI_TRACE=1 LOKI_PIPE_LAG_X10=10000 python tools/one_layer.py --reps 20
LOKI_PIPE_STAGES=3 python tools/one_layer.py --reps 20
LOKI_SPLITK=0 python tools/one_layer.py --reps 20
LOKI_TRACE=1 python tools/one_layer.py --S 32768 --reps 10
