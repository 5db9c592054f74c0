timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
for cfg in "--B 1 --S 32768" "--B 1 --S 16384" "--B 2 --S 8192" "--B 1 --S 4096" "--B 4 --S 32768"; do
  for i in 1 2; do
    echo "cfg[$cfg] head $(LOKI_LIB_PATH=tools/bin/libloki_b200_head.so python tools/one_layer.py $cfg --reps 20 | tail -1)"
    echo "cfg[$cfg] cur  $(python tools/one_layer.py $cfg --reps 20 | tail -1)"
  done
done
