python bench.py --config C3 --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1
python bench.py --config C4 --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1
LOKI_TRACE=1 python tools/one_layer.py --B 32 --H 32 --Hkv 8 --S 32768 --kf 0.125 --df 0.5 --reps 5
