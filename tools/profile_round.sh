#!/bin/bash
# Measurement recipe behind profiles/ (run on a B200 via gpurun; outputs in gpurun_out/):
#   PARTS="benches launches ncu sanitize" (default: all)
#   benches  : bench lines (TGT north-star shape, GQA C3 / C4 / C5s, C1) -- the C2 headline is tools/gpu_session.sh
#   launches : ncu launch lists with DRAM bytes per launch (-> profiles/roofline_traffic.json via
#              tools/traffic_from_launches.py)
#   ncu      : one ncu --set full capture of a C2 layer's pipe launches (split layers: the A and the B launch)
#   sanitize : compute-sanitizer memcheck / synccheck / racecheck on small launches of every plan (tools/sanitize.py)
parts=${PARTS:-"benches launches ncu sanitize"}
mkdir -p gpurun_out
for p in $parts; do
  case $p in
    benches)
      timeout 600 python bench.py --config TGT --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_tgt.json 2> gpurun_out/bench_tgt.err
      timeout 300 python bench.py --config C1 --steps 30 --warmup 5 --no-cpu > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
      timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
      timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
      timeout 900 python bench.py --config C5s --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c5s.json 2> gpurun_out/bench_c5s.err
      for c in tgt c1 c3 c4 c5s; do echo "== $c"; head -c 600 gpurun_out/bench_$c.json; echo; tail -2 gpurun_out/bench_$c.err; done ;;
    launches)
      timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
          -k regex:'pipe_|append_kernel' -c 192 --csv --log-file gpurun_out/launches_c2.csv \
          python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-extras > /dev/null 2>&1
      timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
          -k regex:'pipe_|append_kernel' -c 60 --csv --log-file gpurun_out/launches_tgt.csv \
          python bench.py --config TGT --steps 2 --warmup 3 --no-cpu --no-e2e --no-extras > /dev/null 2>&1
      for c in c3 c4; do
        timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
            -k regex:'pipe_|append_kernel' -c 40 --csv --log-file gpurun_out/launches_$c.csv \
            python bench.py --config ${c^^} --steps 2 --warmup 3 --no-cpu --no-e2e --no-extras > /dev/null 2>&1
      done
      for c in c2 tgt c3 c4; do python tools/traffic_from_launches.py ${c^^} gpurun_out/launches_$c.csv gpurun_out/roofline_traffic.json 2>&1 | tail -12; done ;;
    ncu)
      timeout 900 ncu --set full --import-source on --clock-control none -k regex:'pipe_' -s 60 -c 2 -o gpurun_out/pipe_c2 \
          python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-extras > gpurun_out/ncu_full.log 2>&1
      ncu -i gpurun_out/pipe_c2.ncu-rep --page raw --csv > gpurun_out/pipe_c2_raw.csv 2>&1
      ncu -i gpurun_out/pipe_c2.ncu-rep --page details --csv > gpurun_out/pipe_c2_details.csv 2>&1 ;;
    sanitize)
      for tool in memcheck synccheck racecheck; do
        LOKI_TUNING=1 LOKI_SPIN_S=100000 timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
        echo "sanitizer $tool rc=$?"; tail -4 gpurun_out/sanitize_$tool.log
      done ;;
  esac
done
