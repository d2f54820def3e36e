cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest12.log 2>&1; echo rc=$? >> gpurun_out/gputest12.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1; echo rc=$? >> gpurun_out/g_smoke.log
timeout 900 python bench.py --out gpurun_out/g_sift1m.json > gpurun_out/g_sift1m.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --out gpurun_out/g_ref.json > gpurun_out/g_ref.log 2>&1; echo "ref rc=$?"
