cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_query_gpu.py -x -q 2>&1 | tail -3
for P in 0 20 0 20 12 28; do
  GGNN_PILOT=$P timeout 300 python bench.py --steps 20 --warmup 5 --tau 0.58 --no-cpu-baseline --no-ref-build --out gpurun_out/abp.json > gpurun_out/abp.log 2>&1
  python -c "
import json; j=json.load(open('gpurun_out/abp.json'))
print('P=$P', 'value %.0f kernel %.3f e2e %.0f 2inflight %.0f R@10 %.4f' % (j['value'], j['roofline']['kernel_ms'], j['e2e']['value'], j['details']['two_batches_in_flight']['qps'], j['details']['recall']['R@10']))"
done
