# per-config one-layer timings for halves = 0 / 1 / 2 (mode 0 below 8K rows, split layers from 8K)
for cfg in "--S 4096" "--B 1 --S 4096" "--S 2048" "--Hkv 8 --S 4096" "--B 4 --S 4096" "" "--B 1 --S 8192" "--Hkv 8" "--S 32768" "--Hkv 8 --S 32768"; do
  for h in 0 1 2; do
    echo "cfg[$cfg] halves=$h $(LOKI_PIPE_HALVES=$h python tools/one_layer.py $cfg --reps 20 | tail -1)"
  done
done
for h in 0 1 2; do LOKI_PIPE_HALVES=$h timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --tb=short 2>&1 | tail -1; done
