#!/usr/bin/env bash
# A/B of alternative builds on one workload: WORKLOAD=gist1m tools/gpu_ab_w.sh lib...
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
w=${WORKLOAD:-gist1m}
i=0
for lib in "$@"; do
  i=$((i+1))
  GGNN_LIB=$PWD/$lib timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --tau ${TAU:-0.6} --no-cpu-baseline --no-ref-build \
    --out gpurun_out/abw_$i.json > gpurun_out/abw_$i.log 2>&1
  echo "$lib rc=$?"
  python -c "
import json; j=json.load(open('gpurun_out/abw_$i.json'))
print(' value %.0f kernel %.3f ms frac %.3f build %.1f R@10 %.4f' % (j['value'], j['roofline']['kernel_ms'], j['roofline']['frac'], j['build_seconds'], j['details']['recall']['R@10']))" 2>&1 | tail -1
done
