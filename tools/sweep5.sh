python -m pytest tests -m gpu -x -q 2>&1 | tail -3
LOKI_TRACE=1 python tools/one_layer.py --reps 20
LOKI_PIPE_STAGES=3 python tools/one_layer.py --reps 20
LOKI_PIPE_STAGES=4 python tools/one_layer.py --reps 20
LOKI_PIPE_STAGES=3 LOKI_PIPE_CTAS_PER_SM=3 python tools/one_layer.py --reps 20
LOKI_TRACE=1 python tools/one_layer.py --S 32768 --reps 10
LOKI_PIPE_STAGES=3 python tools/one_layer.py --S 32768 --reps 10
