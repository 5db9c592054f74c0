for la in 1024 2048; do echo "parity LA=$la: $(LOKI_PIPE_LA=$la timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -1)"; done
for cfg in "--B 1 --S 4096" "--B 4 --S 4096" "--S 4096" "--B 2 --S 8192"; do
  for la in 0 512 1024 2048; do echo "cfg[$cfg] LA=$la $(LOKI_PIPE_LA=$la python tools/one_layer.py $cfg --reps 20 | tail -1)"; done
done
