for i in 1 2; do
LOKI_LIB_PATH=tools/bin/libloki_b200_prev.so python tools/one_layer.py --reps 20 | tail -1
python tools/one_layer.py --reps 20 | tail -1
LOKI_SPLITK=0 python tools/one_layer.py --reps 20 | tail -1
done
LOKI_LIB_PATH=tools/bin/libloki_b200_prev.so python tools/one_layer.py --S 32768 --reps 10 | tail -1
python tools/one_layer.py --S 32768 --reps 10 | tail -1
