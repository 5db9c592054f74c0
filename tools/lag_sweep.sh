# split-layer defaults confirmation (C2, TGT, S = 16K, S = 4K) and parity
python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -2
for i in 1 2; do echo c2; python tools/one_layer.py --reps 20 | tail -1; done
echo tgt; python tools/one_layer.py --S 32768 --reps 10 | tail -1
echo s16k; python tools/one_layer.py --S 16384 --reps 10 | tail -1
echo s4k; python tools/one_layer.py --S 4096 --reps 20 | tail -1
echo s4k-comb; LOKI_PIPE_SPLIT=0 python tools/one_layer.py --S 4096 --reps 20 | tail -1
