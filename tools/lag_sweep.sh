# lag (LOKI_PIPE_LAG_X10) sweep for the C5s shard (GQA 8, S = 128K, 128 units)
for l in 200 320 640 2000; do echo c5s-lag$l; LOKI_PIPE_LAG_X10=$l python tools/one_layer.py --B 128 --H 8 --Hkv 1 --S 131072 --reps 3 | tail -1; done
echo c5s-trace; LOKI_TRACE=1 python tools/one_layer.py --B 128 --H 8 --Hkv 1 --S 131072 --reps 2 | grep -v "CTAs in"
