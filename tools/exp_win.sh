cd /root/repo
for w in 1 16 64; do
  echo "== merge windows $w"
  GGNN_MERGE_WINDOWS=$w timeout 300 python -m pytest tests/test_shapes.py -q -s -m gpu -k latent20k 2>&1 | grep "^\[("
  GGNN_MERGE_WINDOWS=$w timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --out gpurun_out/win_$w.json > /dev/null 2>&1
  python -c "
import json;j=json.load(open('gpurun_out/win_$w.json'))
print(' build', round(j['build_seconds'],2), 'tau', j['config']['tau'], 'QPS', round(j['value']), [(r['tau'], r['R@10']) for r in j['config']['tau_sweep']][-4:])"
done
