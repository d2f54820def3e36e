#!/usr/bin/env bash
# A/B of the longest-first schedule (GGNN_PILOT=0 vs default) on other workloads.
# Usage: tools/ab_pilot_w.sh workload [workload ...]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for w in "$@"; do
  for P in 0 20; do
    GGNN_PILOT=$P timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-ref-build \
      --out gpurun_out/abw_${w}_$P.json > gpurun_out/abw_${w}_$P.log 2>&1
    python -c "
import json; j=json.load(open('gpurun_out/abw_${w}_$P.json'))
print('$w P=$P', 'value %.0f kernel %.3f e2e %.0f tau %s R@10 %.4f' % (j['value'], j['roofline']['kernel_ms'], j['e2e']['value'], j['config'].get('tau'), j['details']['recall']['R@10']))" || tail -3 gpurun_out/abw_${w}_$P.log
  done
done
