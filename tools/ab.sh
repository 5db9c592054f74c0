# combined pipe vs split layers (LOKI_PIPE_SPLIT=1), same box
LOKI_PIPE_SPLIT=1 timeout 600 python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -4
for i in 1 2; do
echo comb; python tools/one_layer.py --reps 20 | tail -1
echo split; LOKI_PIPE_SPLIT=1 python tools/one_layer.py --reps 20 | tail -1
done
echo comb-tgt; python tools/one_layer.py --S 32768 --reps 10 | tail -1
echo split-tgt; LOKI_PIPE_SPLIT=1 python tools/one_layer.py --S 32768 --reps 10 | tail -1
echo split-tgt-nobig; LOKI_PIPE_SPLIT=1 LOKI_PIPE_BIG=0 python tools/one_layer.py --S 32768 --reps 10 | tail -1
