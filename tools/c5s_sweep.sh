C5="--B 128 --H 8 --Hkv 1 --S 131072"
for la in 0 4096 16384 32768; do for a in 2 3; do
  echo "C5s LA=$la A_CTAS=$a $(LOKI_PIPE_LA=$la LOKI_PIPE_A_CTAS=$a timeout 300 python tools/one_layer.py $C5 --reps 3 | tail -1)"
done; done
echo "C5s one launch $(LOKI_PIPE_SPLIT=0 timeout 300 python tools/one_layer.py $C5 --reps 3 | tail -1)"
