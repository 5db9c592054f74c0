LOKI_TRACE=1 python tools/one_layer.py --reps 20
LOKI_TRACE=1 LOKI_PIPE_LAG_X10=10000 python tools/one_layer.py --reps 20
LOKI_PIPE_STAGES=2 LOKI_PIPE_STAGE_KB=8 python tools/one_layer.py --reps 20
LOKI_PIPE_STAGES=4 python tools/one_layer.py --reps 20
LOKI_PIPE_STAGES=6 LOKI_PIPE_STAGE_KB=2 python tools/one_layer.py --reps 20
python tools/one_layer.py --reps 20 --mode dense
LOKI_DEBUG=1 python tools/one_layer.py --reps 20 --mode dense
LOKI_PIPE_RP=2048 LOKI_PIPE_LC=8192 python tools/one_layer.py --reps 20
LOKI_PIPE_RP=512 LOKI_PIPE_LC=2048 python tools/one_layer.py --reps 20
