python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -4
LOKI_TRACE=1 python tools/one_layer.py --reps 20
for l in 20 25 30 60; do LOKI_PIPE_LAG_X10=$l python tools/one_layer.py --reps 20; done
LOKI_TRACE=1 python tools/one_layer.py --S 32768 --reps 10
LOKI_PIPE_LAG_X10=25 python tools/one_layer.py --S 32768 --reps 10
