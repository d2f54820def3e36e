#!/usr/bin/env bash
# A/B: GPU tests once, then the bench (fixed tau, no CPU baseline) per library.
# Usage: tools/gpu_ab.sh [lib ...]   (default: the in-tree library only)
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
if [ -z "${SKIP_TESTS:-}" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pytest_gpu.log
fi
libs="${*:-paper_1912_01059_b200/libggnn_b200.so}"
i=0
for lib in $libs; do
  i=$((i+1))
  GGNN_LIB=$PWD/$lib timeout 900 python bench.py --steps 20 --warmup 3 --tau ${TAU:-0.6} --no-cpu-baseline --no-ref-build \
    --out gpurun_out/ab_$i.json > gpurun_out/ab_$i.log 2>&1
  echo "$lib rc=$?"
  python - "$i" <<'PY'
import json, sys
try:
    j = json.load(open(f"gpurun_out/ab_{sys.argv[1]}.json"))
    print(" value %.0f q/s  kernel %.3f ms  build %.2f s  R@10 %.4f  e2e %.0f  2-in-flight %.0f clocks %s" % (
        j["value"], j["roofline"]["kernel_ms"], j["build_seconds"], j["details"]["recall"]["R@10"], j["e2e"]["value"],
        j["details"]["two_batches_in_flight"]["qps"], j["clocks"]))
except Exception as e:
    print(" no result", e)
PY
done
