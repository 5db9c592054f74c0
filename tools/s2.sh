for cfg in "LOKI_PIPE_HALVES=0" "LOKI_PIPE_HALVES=2" "LOKI_PIPE_HALVES=1 LOKI_PIPE_TAIL_X10=2" "LOKI_PIPE_HALVES=1 LOKI_PIPE_TAIL_X10=5" "LOKI_PIPE_HALVES=1 LOKI_PIPE_TAIL_X10=10" "LOKI_PIPE_HALVES=1 LOKI_PIPE_TAIL_X10=20"; do
  echo "=== $cfg"
  env $cfg LOKI_TUNING=1 timeout 120 python tools/one_layer.py --reps 30 2>&1 | grep -v "^plan" | head -3
  env $cfg LOKI_TUNING=1 timeout 120 python tools/one_layer.py --reps 30 --S 32768 2>&1 | grep -v "^plan" | head -3
done
