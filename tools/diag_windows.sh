#!/usr/bin/env bash
# deep3k / gist3k recall of GPU-built graphs for several symmetrize / merge window counts
cd "$(dirname "$0")/.."
for mw in 16 64; do for sw in 16 128; do
  echo "== merge windows $mw, sym windows $sw"
  GGNN_MERGE_WINDOWS=$mw GGNN_SYM_WINDOWS=$sw timeout 300 python tools/diag_deep.py deep3k 2>&1 | grep -E "gpu .*R@1"
done; done
