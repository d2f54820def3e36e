#!/usr/bin/env bash
# Build the committed HEAD sources into paper_1912_01059_b200/lib_old.so and
# the working tree into the in-tree library (A/B pair for tools/gpu_ab.sh).
set -eu
cd "$(dirname "$0")/.."
git stash -q
trap 'git stash pop -q' EXIT
python -c "from paper_1912_01059_b200 import _build_ext as b; b.build(out='paper_1912_01059_b200/lib_old.so')"
git stash pop -q
trap - EXIT
python -c "from paper_1912_01059_b200 import _build_ext as b; b.build()"
