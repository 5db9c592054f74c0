#!/bin/bash
# Same-box A/B (run via gpurun): the working-tree library vs tools/bin/libloki_base.so (the committed HEAD,
# built locally), alternating runs of the given bench configs.  Prints value / attention us per layer.
#   CONFIGS="C2 TGT" REPS=2 tools/ab_run.sh
cfgs=${CONFIGS:-"C2 TGT"}
for r in $(seq ${REPS:-2}); do
  for c in $cfgs; do
    for lib in base new; do
      if [ $lib = base ]; then export LOKI_LIB_PATH=$PWD/tools/bin/libloki_base.so; else unset LOKI_LIB_PATH; fi
      echo -n "$c $lib: "
      timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e --no-extras --no-parity $AB_ARGS 2>/dev/null \
        | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['loki_attention_us_per_layer'], d['roofline']['frac'])"
    done
  done
done
unset LOKI_LIB_PATH
