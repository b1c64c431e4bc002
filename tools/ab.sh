#!/bin/bash
# Same-box A/B of the working tree's library against a saved build (the box-to-box spread is
# +-5 %, so only same-box pairs compare): tools/ab.sh TAG "bench args" [rounds]
#   expects paper_2011_01316_b200/_build/libexpdg_b200_ab.so (the "old" build)
tag=$1; args=$2; rounds=${3:-2}
out=gpurun_out/ab_$tag.log
: > $out
for r in $(seq $rounds); do
  for c in new old; do
    if [ $c = old ]; then export EXPDG_LIB=$PWD/paper_2011_01316_b200/_build/libexpdg_b200_ab.so; else unset EXPDG_LIB; fi
    python bench.py $args --no-cpu-baseline --no-e2e > gpurun_out/ab_${tag}_$c.json 2>>gpurun_out/ab_$tag.err
    python -c "import json;d=json.load(open('gpurun_out/ab_${tag}_$c.json'));r=d['roofline'];print('$c', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], round(r['launch_ms'],4), round(r['achieved']))" >> $out
  done
done
unset EXPDG_LIB
