C3="--B 32 --Hkv 8 --S 32768 --kf 0.125 --df 0.5"; C4="--B 64 --Hkv 8 --S 16384"
for name in C3 C4; do cfg=${!name}
  for la in 0 4096 16384; do for a in 2 3; do
    echo "$name LA=$la A_CTAS=$a $(LOKI_PIPE_LA=$la LOKI_PIPE_A_CTAS=$a python tools/one_layer.py $cfg --reps 5 | tail -1)"
  done; done
  echo "$name halves1 $(LOKI_PIPE_HALVES=1 python tools/one_layer.py $cfg --reps 5 | tail -1)"
done
