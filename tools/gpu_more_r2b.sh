#!/usr/bin/env bash
# Re-measure the remaining workload lines with the final round-2 kernel:
# c1 (both arms), c5 (QPS_1: one GPU searching the 8 shards in turn), deep10m.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python bench.py --workload c1 --steps 10 --out gpurun_out/h_c1.json > gpurun_out/h_c1.log 2>&1; echo "c1 rc=$?"
timeout 600 python bench.py --workload c1 --impl reference --steps 10 --out gpurun_out/h_c1_ref.json > gpurun_out/h_c1_ref.log 2>&1; echo "c1 ref rc=$?"
timeout 2400 python bench.py --workload c5 --steps 10 --no-cpu-baseline --no-ref-build --out gpurun_out/h_c5.json > gpurun_out/h_c5.log 2>&1; echo "c5 rc=$?"
timeout 2400 python bench.py --workload deep10m --steps 5 --no-ref-build --out gpurun_out/h_deep10m.json > gpurun_out/h_deep10m.log 2>&1; echo "deep10m rc=$?"
