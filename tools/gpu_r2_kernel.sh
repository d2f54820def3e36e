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
        python bench.py --steps 3 --warmup 3 --tau 0.58 --no-cpu-baseline --no-ref-build > gpurun_out/launches.log 2>&1; echo "launches rc=$?" ;;
    ncu) timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
        -k regex:_ZN4ggnn12query_kernelIhhLi8ELb0ELb0E -s 6 -c 1 -f -o gpurun_out/query_full \
        python bench.py --steps 2 --warmup 3 --tau 0.58 --no-cpu-baseline --no-ref-build > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?" ;;
    torchrun)
      GGNN_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --workload c5 --points 800000 --steps 10 --warmup 3 --out gpurun_out/b_c5mini2.json > gpurun_out/b_c5mini2.log 2>&1; echo "c5mini2 rc=$?"
      GGNN_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus 2 --steps 10 --warmup 3 --points 200000 --out gpurun_out/b_repl2.json > gpurun_out/b_repl2.log 2>&1; echo "repl2 rc=$?"
      timeout 600 python bench.py --workload c5 --points 800000 --steps 10 --warmup 3 --no-cpu-baseline --out gpurun_out/b_c5mini.json > gpurun_out/b_c5mini.log 2>&1; echo "c5mini rc=$?"
      for f in gpurun_out/b_c5mini2.log gpurun_out/b_repl2.log gpurun_out/b_c5mini.log; do echo "== $f"; tail -c 600 $f; echo; done ;;
    swap) timeout 900 python -m pytest tests/test_backend_swap_gpu.py -m gpu -q > gpurun_out/pytest_swap.log 2>&1; echo "swap rc=$?"; tail -3 gpurun_out/pytest_swap.log ;;
    bq) timeout 900 python tools/batch_query_probe.py > gpurun_out/bq.log 2>&1; echo "bq rc=$?"; cat gpurun_out/bq.log | tail -5 ;;
    leaf) for k in gist deep; do timeout 600 python tools/leaf_probe.py $k 200000; done > gpurun_out/leaf.log 2>&1; echo "leaf rc=$?"; cat gpurun_out/leaf.log
          timeout 900 ncu --set full --clock-control none --kernel-name-base mangled -k regex:leaf_knn_tf32 -c 1 -f -o gpurun_out/leaf_tf32 python tools/leaf_probe.py gist 200000 > gpurun_out/leaf_ncu.log 2>&1; echo "leaf ncu rc=$?" ;;
    workloads) for w in sift1m-f32 gist1m; do timeout 1500 python bench.py --workload $w --steps 10 --warmup 3 --no-ref-build --out gpurun_out/b_$w.json > gpurun_out/b_$w.log 2>&1; echo "$w rc=$?"; tail -c 400 gpurun_out/b_$w.log; echo; done ;;
    long) free -g; nproc
          timeout 1800 python bench.py --workload deep10m --steps 10 --warmup 3 --no-ref-build --out gpurun_out/b_deep10m.json > gpurun_out/b_deep10m.log 2>&1; echo "deep10m rc=$?"; tail -c 300 gpurun_out/b_deep10m.log; echo
          timeout 3000 python bench.py --workload c5 --steps 10 --warmup 3 --out gpurun_out/b_c5.json > gpurun_out/b_c5.log 2>&1; echo "c5 rc=$?"; tail -c 300 gpurun_out/b_c5.log; echo ;;
    c1) timeout 900 python bench.py --workload c1 --steps 10 --warmup 3 --out gpurun_out/b_c1.json > gpurun_out/b_c1.log 2>&1; echo "c1 rc=$?"
        timeout 900 python bench.py --workload c1 --impl reference --steps 3 --warmup 1 --out gpurun_out/b_c1_ref.json > gpurun_out/b_c1_ref.log 2>&1; echo "c1 ref rc=$?"; tail -c 400 gpurun_out/b_c1_ref.log; echo ;;
    ncuw) for w in sift1m-f32 gist1m; do
            timeout 1500 ncu --set full --clock-control none --kernel-name-base mangled -k regex:_ZN4ggnn12query_kernelIffLi -s 6 -c 1 -f \
              -o gpurun_out/query_$w python bench.py --workload $w --steps 2 --warmup 3 --tau 0.6 --no-cpu-baseline --no-ref-build > gpurun_out/ncu_$w.log 2>&1; echo "ncu $w rc=$?"; done ;;
  esac
done
