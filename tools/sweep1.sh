set -x
for c in 1 2 4 8; do LOKI_CLUSTER=$c python tools/one_layer.py --reps 20; done
for kb in 72 80 96 140; do LOKI_SMEM_KB=$kb python tools/one_layer.py --reps 20; done
LOKI_SMEM_KB=72 LOKI_CLUSTER=4 python tools/one_layer.py --reps 20
LOKI_TRACE=1 python tools/one_layer.py --reps 20
python tools/one_layer.py --S 32768 --reps 10
LOKI_TRACE=1 python tools/one_layer.py --S 32768 --reps 10
python tools/one_layer.py --S 32768 --reps 10 --mode dense
python tools/one_layer.py --reps 10 --mode dense
