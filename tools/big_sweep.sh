for S in 8192 16384; do
for big in 0 1; do for h in 0 1; do
  echo "S=$S BIG=$big HALVES=$h $(LOKI_PIPE_BIG=$big LOKI_PIPE_HALVES=$h python tools/one_layer.py --S $S --reps 20 | tail -1)"
done; done; done
echo "C4 default $(python tools/one_layer.py --B 64 --Hkv 8 --S 16384 --reps 10 | tail -1)"
echo "C4 halves2 $(LOKI_PIPE_HALVES=2 python tools/one_layer.py --B 64 --Hkv 8 --S 16384 --reps 10 | tail -1)"
echo "C4 halves1 $(LOKI_PIPE_HALVES=1 python tools/one_layer.py --B 64 --Hkv 8 --S 16384 --reps 10 | tail -1)"
