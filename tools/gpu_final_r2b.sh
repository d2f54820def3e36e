#!/usr/bin/env bash
# Final measurement session of round 2 (second half): smoke, the default bench
# line (the driver's command), sift1m-f32 / c5shard / gist1m lines, one full
# ncu capture of a scheduled C2 batch and the ncu launch list of the bench
# command.  Stages: smoke bench f32 c5shard gist ncu launches (default: all).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
stages="${*:-smoke bench f32 c5shard gist ncu launches}"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_info.csv 2>&1
for s in $stages; do
  case $s in
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?" ;;
    bench)
      timeout 900 python bench.py --out gpurun_out/f_sift1m.json > gpurun_out/f_sift1m.log 2>&1; echo "bench rc=$?" ;;
    f32)
      timeout 900 python bench.py --workload sift1m-f32 --out gpurun_out/f_sift1m_f32.json > gpurun_out/f_sift1m_f32.log 2>&1; echo "f32 rc=$?" ;;
    c5shard)
      timeout 1200 python bench.py --workload c5shard --no-cpu-baseline --no-ref-build --out gpurun_out/f_c5shard.json > gpurun_out/f_c5shard.log 2>&1; echo "c5shard rc=$?" ;;
    gist)
      timeout 1500 python bench.py --workload gist1m --out gpurun_out/f_gist1m.json > gpurun_out/f_gist1m.log 2>&1; echo "gist rc=$?" ;;
    ncu)
      timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -f \
        -o gpurun_out/f_sched_full python tools/ncu_sched.py > gpurun_out/f_ncu_sched.log 2>&1; echo "ncu rc=$?" ;;
    launches)
      timeout 2700 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv \
        python bench.py --steps 3 --warmup 3 --tau 0.58 --no-cpu-baseline --no-ref-build > gpurun_out/f_launches.log 2>&1
      echo "launches rc=$?"; gzip -f gpurun_out/f_launches.csv ;;
  esac
done
