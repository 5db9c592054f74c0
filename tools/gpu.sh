#!/bin/bash
# Build locally (abort on failure), then run the given command on a B200 via gpurun.
#   tools/gpu.sh <timeout_s> '<command>'
set -e
cd "$(dirname "$0")/.."
python -m paper_2406_02542_b200._build > /tmp/loki_build.log 2>&1 || { tail -20 /tmp/loki_build.log; echo "BUILD FAILED"; exit 1; }
exec /usr/local/graft/bin/gpurun --timeout "$1" -- "$2"
