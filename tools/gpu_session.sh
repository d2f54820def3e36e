#!/usr/bin/env bash
# One gpurun session: GPU tests, smoke, bench, ncu launch list and one full
# capture of the query kernel.  Usage: tools/gpu_session.sh [stage ...]
# stages: tests smoke bench launches ncu   (default: all)
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
stages="${*:-tests smoke bench launches ncu}"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_info.csv 2>&1
for s in $stages; do
  case $s in
    tests)
      timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "tests rc=$?" ;;
    smoke)
      timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" ;;
    bench)
      timeout 1200 python bench.py --steps 20 --warmup 3 --out gpurun_out/bench.json > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.log ;;
    launches)
      timeout 2700 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
        python bench.py --steps 3 --warmup 3 --tau ${TAU:-0.55} --no-cpu-baseline > gpurun_out/launches.log 2>&1; echo "launches rc=$?" ;;
    ncu)
      timeout 1500 ncu --set full --clock-control none --import-source on -k regex:query_kernel -s 2 -c 1 -f \
        -o gpurun_out/query_full python bench.py --steps 1 --warmup 3 --tau ${TAU:-0.55} --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?" ;;
  esac
done
