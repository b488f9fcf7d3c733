#!/bin/bash
# time every K3 tiling variant on one config: tools/sweep_variants.sh n p pop
for v in 0 1 2 3 4 5 6 7 8; do
  echo -n "variant $v: "
  HUBGPU_FIT_VARIANT=$v python tools/prof_fitness.py "$@" 2>&1 | tail -1
done
