# lag (LOKI_PIPE_LAG_X10) sweep for the GQA shapes
for l in 50 70 100; do echo c3lag$l; LOKI_PIPE_LAG_X10=$l python tools/one_layer.py --B 32 --H 32 --Hkv 8 --S 32768 --kf 0.125 --df 0.5 --reps 5 | tail -1; done
for l in 50 70 100 160; do echo c4lag$l; LOKI_PIPE_LAG_X10=$l python tools/one_layer.py --B 64 --H 32 --Hkv 8 --S 16384 --kf 0.25 --df 0.25 --reps 5 | tail -1; done
