#!/bin/bash
# A/B per-kernel timing of libdbp tuning variants: scripts/ab_libs.sh "cg admm bf" build_var/*.so
solvers=$1; shift
for lib in "$@"; do
  for s in $solvers; do echo -n "$(basename $lib) "; DBP_LIB=$PWD/$lib python scripts/time_kernels.py --solver $s; done
done
