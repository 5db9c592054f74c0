python -m pytest tests -m gpu -x -q 2>&1 | tail -15
LOKI_TRACE=1 python tools/one_layer.py --reps 20
LOKI_PIPE=0 python tools/one_layer.py --reps 20
LOKI_SPLITK=0 python tools/one_layer.py --reps 20
LOKI_PIPE_STAGES=2 python tools/one_layer.py --reps 20
LOKI_TRACE=1 python tools/one_layer.py --S 32768 --reps 10
