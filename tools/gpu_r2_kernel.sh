#!/usr/bin/env bash
# Round-2 kernel check: GPU tests, a short bench, the launch list and one full
# ncu capture of the benchmarked query kernel (sift1m).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
stages="${*:-tests bench ncu}"
for s in $stages; do
  case $s in
    tests) timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pytest_gpu.log ;;
    bench) timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-ref-build --out gpurun_out/b_quick.json > gpurun_out/b_quick.log 2>&1; echo "bench rc=$?"
           python -c "import json;d=json.load(open('gpurun_out/b_quick.json'));print(d['value'],d['e2e']['value'],d['roofline']['kernel_ms'],d['details']['two_batches_in_flight']['qps'],d['details']['recall'])" ;;
    launches) timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
        python bench.py --steps 3 --warmup 3 --tau 0.6 --no-cpu-baseline --no-ref-build > gpurun_out/launches.log 2>&1; echo "launches rc=$?" ;;
    ncu) timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
        -k regex:_ZN4ggnn12query_kernelIhhLi8ELb0ELb0E -s 6 -c 1 -f -o gpurun_out/query_full \
        python bench.py --steps 2 --warmup 3 --tau 0.6 --no-cpu-baseline --no-ref-build > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?" ;;
    torchrun)
      GGNN_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --workload c5 --points 800000 --steps 10 --warmup 3 --out gpurun_out/b_c5mini2.json > gpurun_out/b_c5mini2.log 2>&1; echo "c5mini2 rc=$?"
      GGNN_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus 2 --steps 10 --warmup 3 --points 200000 --out gpurun_out/b_repl2.json > gpurun_out/b_repl2.log 2>&1; echo "repl2 rc=$?"
      timeout 600 python bench.py --workload c5 --points 800000 --steps 10 --warmup 3 --no-cpu-baseline --out gpurun_out/b_c5mini.json > gpurun_out/b_c5mini.log 2>&1; echo "c5mini rc=$?"
      for f in gpurun_out/b_c5mini2.log gpurun_out/b_repl2.log gpurun_out/b_c5mini.log; do echo "== $f"; tail -c 600 $f; echo; done ;;
  esac
done
