#!/usr/bin/env bash
# A/B of the longest-first schedule settings on the C2 bench (fixed tau).
# Usage: tools/ab_pilot.sh "P1 P2 A" ["P1 P2 A" ...]   (P1 = 0: plain launch)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for cfg in "$@"; do
  set -- $cfg
  GGNN_PILOT=$1 GGNN_PILOT2=$2 GGNN_PILOT_A=$3 timeout 300 python bench.py --steps 20 --warmup 5 --tau 0.58 \
    --no-cpu-baseline --no-ref-build --out gpurun_out/abp.json > gpurun_out/abp.log 2>&1
  python -c "
import json; j=json.load(open('gpurun_out/abp.json'))
print('$cfg', 'value %.0f kernel %.3f e2e %.0f %s 2inflight %.0f R@10 %.4f' % (j['value'], j['roofline']['kernel_ms'], j['e2e']['value'], j['e2e'].get('call_ms'), j['details']['two_batches_in_flight']['qps'], j['details']['recall']['R@10']))" || tail -3 gpurun_out/abp.log
done
