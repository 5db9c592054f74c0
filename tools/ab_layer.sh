# same-box A/B of one layer (tools/one_layer.py) between the committed library and the working tree
for cfg in "" "--S 32768" "--S 16384" "--B 64 --Hkv 8 --S 16384" "--S 4096"; do
  for i in 1 2; do
    echo "cfg[$cfg] head $(LOKI_LIB_PATH=tools/bin/libloki_b200_head.so python tools/one_layer.py $cfg --reps 20 | tail -1)"
    echo "cfg[$cfg] cur  $(python tools/one_layer.py $cfg --reps 20 | tail -1)"
  done
done
echo "C2 B_STAGES=2 $(LOKI_PIPE_B_STAGES=2 python tools/one_layer.py --reps 20 | tail -1)"
echo "C2 B_STAGES=4 $(LOKI_PIPE_B_STAGES=4 python tools/one_layer.py --reps 20 | tail -1)"
