python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -25
LOKI_TRACE=1 python tools/one_layer.py --reps 20
LOKI_PIPE_MMA=0 python tools/one_layer.py --reps 20
LOKI_PIPE_STAGES=3 python tools/one_layer.py --reps 20
LOKI_TRACE=1 python tools/one_layer.py --S 32768 --reps 10
