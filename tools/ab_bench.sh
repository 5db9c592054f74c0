# same-box A/B of the full C2 step (K0 + pipe per layer) between the committed library and the working tree
for i in 1 2; do
echo head; LOKI_LIB_PATH=tools/bin/libloki_b200_head.so python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e --no-extras 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(j['value'], j['loki_attention_us_per_layer'])"
echo cur; python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e --no-extras 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(j['value'], j['loki_attention_us_per_layer'])"
done
