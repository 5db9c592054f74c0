#!/bin/bash
# Round-end evidence session (run via gpurun from the repo root): GPU tests, smoke, the default bench line, then
# tools/profile_round.sh benches + launch lists + ncu captures (compute-sanitizer is closed on the pool).
# Outputs in gpurun_out/.
set -x
timeout 1200 python -m pytest tests -m gpu -q --tb=short -x > gpurun_out/tests_gpu.log 2>&1; tail -2 gpurun_out/tests_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -c 400 gpurun_out/bench_c2.json
PARTS=${ROUND_PARTS:-"benches launches ncu"} bash tools/profile_round.sh
