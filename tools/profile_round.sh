#!/bin/bash
# Measurement recipe behind profiles/ (run on a B200 via gpurun; outputs in gpurun_out/):
#   PARTS="benches launches ncu sanitize" (default: all)
#   benches  : bench lines (TGT north-star shape, C1, GQA C3 / C4 / C5s per-head and group-shared) -- the C2
#              headline is `python bench.py` itself
#   launches : ncu launch lists with DRAM bytes per launch (-> roofline_traffic.json via
#              tools/traffic_from_launches.py)
#   ncu      : ncu --set full captures of a C2 layer (K0, the A launch, the B launch) and a C3 per-head layer
#   sanitize : compute-sanitizer memcheck / synccheck / racecheck on small launches of every plan (tools/sanitize.py)
parts=${PARTS:-"benches launches ncu sanitize"}
mkdir -p gpurun_out
line() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['loki_attention_us_per_layer'], d.get('speedup_vs_best_dense'), d['roofline']['frac'], (d.get('parity') or {}).get('pass'))"; }
for p in $parts; do
  case $p in
    benches)
      timeout 600 python bench.py --config TGT --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_tgt.json 2> gpurun_out/bench_tgt.err
      timeout 300 python bench.py --config C1 --steps 30 --warmup 5 --no-cpu > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
      for c in C3 C4 C5s; do
        for gs in per_head shared; do
          timeout 900 python bench.py --config $c --group-select $gs --steps 5 --warmup 3 --no-cpu --no-e2e \
              > gpurun_out/bench_${c,,}_$gs.json 2> gpurun_out/bench_${c,,}_$gs.err
        done
      done
      for f in gpurun_out/bench_tgt.json gpurun_out/bench_c1.json gpurun_out/bench_c[345]*_*.json; do echo "== $f"; line < $f; done ;;
    launches)
      timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
          -k regex:'pipe_|append_kernel' -c 192 --csv --log-file gpurun_out/launches_c2.csv \
          python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-extras --no-parity > /dev/null 2>&1
      timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
          -k regex:'pipe_|append_kernel' -c 60 --csv --log-file gpurun_out/launches_tgt.csv \
          python bench.py --config TGT --steps 2 --warmup 3 --no-cpu --no-e2e --no-extras --no-parity > /dev/null 2>&1
      for c in C3 C4; do
        for gs in per_head shared; do
          timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
              -k regex:'pipe_|append_kernel' -c 40 --csv --log-file gpurun_out/launches_${c,,}_$gs.csv \
              python bench.py --config $c --group-select $gs --steps 2 --warmup 3 --no-cpu --no-e2e --no-extras --no-parity > /dev/null 2>&1
        done
      done
      python tools/traffic_from_launches.py C2 gpurun_out/launches_c2.csv gpurun_out/roofline_traffic.json | tail -4
      python tools/traffic_from_launches.py TGT gpurun_out/launches_tgt.csv gpurun_out/roofline_traffic.json | tail -4
      for c in c3 c4; do for gs in per_head shared; do
        python tools/traffic_from_launches.py ${c^^}_$gs gpurun_out/launches_${c}_$gs.csv gpurun_out/roofline_traffic.json | tail -4
      done; done ;;
    ncu)
      timeout 900 ncu --set full --import-source on --clock-control none -k regex:'pipe_|append_kernel' -s 9 -c 3 -o gpurun_out/c2_layer \
          python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-extras --no-parity > gpurun_out/ncu_c2.log 2>&1
      ncu -i gpurun_out/c2_layer.ncu-rep --page raw --csv > gpurun_out/c2_layer_raw.csv 2>&1
      timeout 900 ncu --set full --import-source on --clock-control none -k regex:'pipe_' -s 6 -c 2 -o gpurun_out/c3_layer \
          python bench.py --config C3 --steps 2 --warmup 3 --no-cpu --no-e2e --no-extras --no-parity > gpurun_out/ncu_c3.log 2>&1
      ncu -i gpurun_out/c3_layer.ncu-rep --page raw --csv > gpurun_out/c3_layer_raw.csv 2>&1 ;;
    sanitize)
      for tool in memcheck synccheck racecheck; do
        LOKI_TUNING=1 LOKI_SPIN_S=100000 timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
        echo "sanitizer $tool rc=$?"; tail -2 gpurun_out/sanitize_$tool.log
      done ;;
  esac
done
