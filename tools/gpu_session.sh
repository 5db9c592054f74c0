#!/bin/bash
# One measurement session on a B200 (run via gpurun from the repo root): GPU tests, the default bench line,
# the reference arm, and compute-sanitizer on small pipe-kernel launches.  Outputs in gpurun_out/.
#   SESSION_PARTS="tests bench ref sanitize" (default: all)
parts=${SESSION_PARTS:-"tests bench ref sanitize"}
mkdir -p gpurun_out
for p in $parts; do
  case $p in
    tests) timeout 1500 python -m pytest tests -m gpu -q --tb=short -x > gpurun_out/tests_gpu.log 2>&1; tail -3 gpurun_out/tests_gpu.log ;;
    bench) timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.json; tail -3 gpurun_out/bench.err ;;
    ref) timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json | head -c 1500; tail -3 gpurun_out/bench_ref.err ;;
    sanitize)
      for tool in memcheck synccheck racecheck; do
        LOKI_TUNING=1 LOKI_SPIN_S=100000 timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
        echo "sanitizer $tool rc=$?"; tail -4 gpurun_out/sanitize_$tool.log
      done ;;
  esac
done
