#!/usr/bin/env bash
cd "$(dirname "$0")/.."
for w in 16 64 256 1024; do echo "== windows $w"; GGNN_SYM_WINDOWS=$w timeout 300 python tools/diag_deep.py deep3k 2>&1 | grep -E "C@10|sym used|tau 0.6|tau 2.0"; done
