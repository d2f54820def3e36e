set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_info.csv 2>&1
timeout 900 python bench.py --steps 20 --warmup 3 --out gpurun_out/b_sift1m.json > gpurun_out/b_sift1m.log 2>&1; echo "sift1m rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 --out gpurun_out/b_ref.json > gpurun_out/b_ref.log 2>&1; echo "ref rc=$?"
timeout 600 python bench.py --workload c5 --points 800000 --steps 10 --warmup 3 --no-cpu-baseline --out gpurun_out/b_c5mini.json > gpurun_out/b_c5mini.log 2>&1; echo "c5mini rc=$?"
GGNN_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --workload c5 --points 800000 --steps 10 --warmup 3 --out gpurun_out/b_c5mini2.json > gpurun_out/b_c5mini2.log 2>&1; echo "c5mini2 rc=$?"
GGNN_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus 2 --steps 10 --warmup 3 --points 200000 --out gpurun_out/b_repl2.json > gpurun_out/b_repl2.log 2>&1; echo "repl2 rc=$?"
for f in gpurun_out/b_*.log; do echo "== $f"; tail -c 1500 $f; echo; done
