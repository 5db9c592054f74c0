#!/bin/bash
# Tuning sweep (run via gpurun): bench lines under LOKI_TUNING knob settings.
#   tools/knob_sweep.sh "<config> <bench args>" "<KNOB=v ...>" ["<KNOB=v ...>" ...]
spec=$1; shift
for kv in "$@"; do
  echo -n "$spec [$kv]: "
  env LOKI_TUNING=1 $kv timeout 300 python bench.py --config $spec --steps ${STEPS:-20} --warmup 5 --no-cpu --no-e2e --no-extras --no-parity 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['loki_attention_us_per_layer'])"
done
