timeout 900 python -m pytest tests -m gpu -q --tb=short 2>&1 | tail -5
for cfg in "--S 4096" "--B 1 --S 4096" "--Hkv 8 --S 4096" "--B 4 --S 4096"; do echo "cfg[$cfg] $(python tools/one_layer.py $cfg --reps 20 | tail -1)"; done
