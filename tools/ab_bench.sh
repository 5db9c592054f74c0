# same-box A/B of the full C2 / TGT step (K0 + pipe per layer) between the committed library and the working tree
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for i in 1 2; do
for cfg in C2 TGT; do
echo "$cfg head $(LOKI_LIB_PATH=tools/bin/libloki_b200_head.so python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu --no-e2e --no-extras 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(j['value'], j['loki_attention_us_per_layer'], j['append_us_per_layer'])")"
echo "$cfg cur  $(python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu --no-e2e --no-extras 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(j['value'], j['loki_attention_us_per_layer'], j['append_us_per_layer'])")"
done
done
