# split-layer knobs at C2 (S = 8K) and TGT (S = 32K): A CTAs per SM x A chunk rows
for S in 8192 32768; do
  for a in 1 2 3; do
    for la in 4096 8192 16384; do
      echo "S=$S A_CTAS=$a LA=$la $(LOKI_PIPE_A_CTAS=$a LOKI_PIPE_LA=$la python tools/one_layer.py --S $S --reps 20 | tail -1)"
    done
  done
  for t in 1 2 4; do echo "S=$S tail halves x10=$t $(LOKI_PIPE_HALVES=1 LOKI_PIPE_TAIL_X10=$t python tools/one_layer.py --S $S --reps 20 | tail -1)"; done
done
