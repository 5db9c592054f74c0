for i in 1 2; do
for la in 0 16384 32768; do echo "TGT LA=$la $(LOKI_PIPE_LA=$la python tools/one_layer.py --S 32768 --reps 10 | tail -1)"; done
for la in 0 16384; do echo "C4 LA=$la $(LOKI_PIPE_LA=$la python tools/one_layer.py --B 64 --Hkv 8 --S 16384 --reps 5 | tail -1)"; done
done
