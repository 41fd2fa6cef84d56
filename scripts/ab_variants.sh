#!/bin/bash
# A/B the build_var/*.so variants: per-kernel device times of the three solvers on configs C/D.
# usage (on the GPU box): bash scripts/ab_variants.sh v0 v1 ... > gpurun_out/ab.txt
for v in "$@"; do
  for s in admm bf cg; do
    cfg=C; [ $s = bf ] && cfg=D
    echo "$v $(DBP_LIB=build_var/$v.so python scripts/time_kernels.py --solver $s --config $cfg --reps 30 2>&1 | tail -1)"
  done
done
