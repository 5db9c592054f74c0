# same-box A/B of the committed library (tools/bin/libloki_b200_head.so) against the working tree
python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -3
for i in 1 2; do
echo head; LOKI_LIB_PATH=tools/bin/libloki_b200_head.so python tools/one_layer.py --reps 20 | tail -1
echo cur; python tools/one_layer.py --reps 20 | tail -1
done
echo head-tgt; LOKI_LIB_PATH=tools/bin/libloki_b200_head.so python tools/one_layer.py --S 32768 --reps 10 | tail -1
echo cur-tgt; python tools/one_layer.py --S 32768 --reps 10 | tail -1
echo head-c3; LOKI_LIB_PATH=tools/bin/libloki_b200_head.so python tools/one_layer.py --B 32 --H 32 --Hkv 8 --S 32768 --kf 0.125 --df 0.5 --reps 5 | tail -1
echo cur-c3; python tools/one_layer.py --B 32 --H 32 --Hkv 8 --S 32768 --kf 0.125 --df 0.5 --reps 5 | tail -1
