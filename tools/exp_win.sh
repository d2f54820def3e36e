#!/usr/bin/env bash
# 1M build time / recall for merge-window and sym-window settings: tools/exp_win.sh "16:16 16:128 32:128"
cd "$(dirname "$0")/.."
for cfg in ${1:-16:16 16:128}; do
  mw=${cfg%%:*}; sw=${cfg##*:}
  GGNN_MERGE_WINDOWS=$mw GGNN_SYM_WINDOWS=$sw timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --out gpurun_out/win_${mw}_${sw}.json > /dev/null 2>&1
  python -c "
import json;j=json.load(open('gpurun_out/win_${mw}_${sw}.json'))
print('merge $mw sym $sw: build', round(j['build_seconds'],2), 'tau', j['config']['tau'], 'QPS', round(j['value']), [(r['tau'], r['R@10']) for r in j['config']['tau_sweep']][-3:])"
done
