python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -3
for i in 1 2; do
echo prev; LOKI_LIB_PATH=tools/bin/libloki_b200_prev.so python tools/one_layer.py --reps 20 | tail -1
echo cur; python tools/one_layer.py --reps 20 | tail -1
echo cur-nosplit; LOKI_SPLITK=0 python tools/one_layer.py --reps 20 | tail -1
done
echo prev-tgt; LOKI_LIB_PATH=tools/bin/libloki_b200_prev.so python tools/one_layer.py --S 32768 --reps 10 | tail -1
echo cur-tgt; python tools/one_layer.py --S 32768 --reps 10 | tail -1
echo prev-c3; LOKI_LIB_PATH=tools/bin/libloki_b200_prev.so python tools/one_layer.py --B 32 --H 32 --Hkv 8 --S 32768 --kf 0.125 --df 0.5 --reps 5 | tail -1
echo cur-c3; python tools/one_layer.py --B 32 --H 32 --Hkv 8 --S 32768 --kf 0.125 --df 0.5 --reps 5 | tail -1
