#!/usr/bin/env bash
# Quick kernel A/B on the C2 workload: build time + query-kernel time at 10k
# and 20k queries per library, libraries interleaved twice (noise check).
# Usage: tools/ab_quick.sh lib_a.so lib_b.so ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
  for lib in "$@"; do
    echo "== $lib (rep $rep)"
    GGNN_LIB=$PWD/$lib timeout 300 python tools/latency_probe.py ${TAU:-0.58} ${SIZES:-10000,20000} 2>&1 | grep -v "^flags"
  done
done
