#!/usr/bin/env bash
# Full ncu capture of one query-kernel launch of the bench workload (1 GPU).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-query_kernel} -s ${SKIP:-2} -c 1 -f \
  -o gpurun_out/${OUT:-query_full} python bench.py --steps 1 --warmup 3 --tau ${TAU:-0.55} --no-cpu-baseline \
  > gpurun_out/ncu_${OUT:-query_full}.log 2>&1
echo "ncu rc=$?"
