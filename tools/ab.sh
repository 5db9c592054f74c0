# same-box A/B of the committed library (tools/bin/libloki_b200_head.so) against the working tree
python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -3
echo head; LOKI_LIB_PATH=tools/bin/libloki_b200_head.so python tools/one_layer.py --reps 20 | tail -1
echo cur; python tools/one_layer.py --reps 20 | tail -1
echo head-c3; LOKI_LIB_PATH=tools/bin/libloki_b200_head.so python tools/one_layer.py --B 32 --H 32 --Hkv 8 --S 32768 --kf 0.125 --df 0.5 --reps 5 | tail -1
echo cur-c3; python tools/one_layer.py --B 32 --H 32 --Hkv 8 --S 32768 --kf 0.125 --df 0.5 --reps 5 | tail -1
echo head-c4; LOKI_LIB_PATH=tools/bin/libloki_b200_head.so python tools/one_layer.py --B 64 --H 32 --Hkv 8 --S 16384 --kf 0.25 --df 0.25 --reps 5 | tail -1
echo cur-c4; python tools/one_layer.py --B 64 --H 32 --Hkv 8 --S 16384 --kf 0.25 --df 0.25 --reps 5 | tail -1
echo head-c5s; LOKI_LIB_PATH=tools/bin/libloki_b200_head.so python tools/one_layer.py --B 128 --H 8 --Hkv 1 --S 131072 --reps 3 | tail -1
echo cur-c5s; python tools/one_layer.py --B 128 --H 8 --Hkv 1 --S 131072 --reps 3 | tail -1
