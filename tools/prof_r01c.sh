python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -3
python bench.py --steps 30 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --config TGT --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_tgt.json 2> gpurun_out/bench_tgt.err
python -c "
import json
for f in ['gpurun_out/bench_c2.json', 'gpurun_out/bench_tgt.json']:
    j = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, j['value'], j['loki_attention_us_per_layer'], j['roofline']['achieved'], j['roofline']['frac'], j.get('speedup_vs_best_dense_attention'), j['speedup_vs_dense_attention_only'], j['e2e']['value'] if j['e2e'] else None)
"
