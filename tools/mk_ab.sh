#!/bin/bash
# Builds HEAD's library as the A/B baseline (libexpdg_b200_ab.so), then the working tree's.
set -e
cd "$(dirname "$0")/.."
git stash -q
python -c "from paper_2011_01316_b200 import _build; _build.build()" 2>&1 | grep -i error || true
cp paper_2011_01316_b200/_build/libexpdg_b200.so paper_2011_01316_b200/_build/libexpdg_b200_ab.so
git stash pop -q
python -c "from paper_2011_01316_b200 import _build; _build.build()" 2>&1 | grep -i error || true
