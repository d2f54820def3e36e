#!/usr/bin/env bash
# float-data A/B: float parity tests + gist1m bench per library
cd "$(dirname "$0")/.."
for lib in ${*:-paper_1912_01059_b200/libggnn_b200.so}; do
  echo "== $lib"
  GGNN_LIB=$PWD/$lib timeout 600 python -m pytest tests/test_shapes.py tests/test_query_gpu.py -q -m gpu -k "float or shapes or gist or deep" 2>&1 | tail -2
  GGNN_LIB=$PWD/$lib timeout 900 python bench.py --workload gist1m --steps 5 --warmup 3 --tau 0.7 --no-cpu-baseline --out gpurun_out/g.json > /dev/null 2>&1
  python -c "
import json;j=json.load(open('gpurun_out/g.json'))
print(' gist1m QPS', round(j['value']), 'kernel ms', round(j['roofline']['kernel_ms'],2), 'R@10', j['config']['recall']['R@10'], 'build', round(j['build_seconds'],1), 'frac', round(j['roofline']['frac'],3))"
done
