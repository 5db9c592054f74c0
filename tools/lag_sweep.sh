# TGT chunking sweep (host knobs only): A chunk rows x B part rows x split-K
for i in 1 2; do
echo big; python tools/one_layer.py --S 32768 --reps 10 | tail -1
echo la8192; LOKI_PIPE_BIG=0 LOKI_PIPE_LA=8192 python tools/one_layer.py --S 32768 --reps 10 | tail -1
echo la8192-split; LOKI_PIPE_BIG=0 LOKI_PIPE_LA=8192 LOKI_SPLITK=1 python tools/one_layer.py --S 32768 --reps 10 | tail -1
echo la16384; LOKI_PIPE_BIG=0 LOKI_PIPE_LA=16384 python tools/one_layer.py --S 32768 --reps 10 | tail -1
echo big-la16384; LOKI_PIPE_LA=16384 python tools/one_layer.py --S 32768 --reps 10 | tail -1
done
