# defaults: split layers for all bf16 S >= 8192, no half parts
python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -2
LOKI_PIPE_SPLIT=1 python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -2
echo c2; python tools/one_layer.py --reps 20 | tail -1
echo tgt; python tools/one_layer.py --S 32768 --reps 10 | tail -1
echo c3; python tools/one_layer.py --B 32 --H 32 --Hkv 8 --S 32768 --kf 0.125 --df 0.5 --reps 5 | tail -1
echo c4; python tools/one_layer.py --B 64 --H 32 --Hkv 8 --S 16384 --kf 0.25 --df 0.25 --reps 5 | tail -1
echo s4k; python tools/one_layer.py --S 4096 --reps 20 | tail -1
