for cfg in "LOKI_SPLITK=0 LOKI_SELECT_WS=0" "LOKI_SPLITK=1"; do
  echo "=== $cfg"
  for S in 8192; do env $cfg LOKI_TUNING=1 LOKI_TRACE=1 timeout 120 python tools/one_layer.py --reps 20 --S $S 2>&1 | grep -v "^plan" | head -6; done
  for S in 32768; do env $cfg LOKI_PIPE_BIG=0 LOKI_TUNING=1 LOKI_TRACE=1 timeout 120 python tools/one_layer.py --reps 20 --S $S 2>&1 | grep -v "^plan" | head -6; done
done
