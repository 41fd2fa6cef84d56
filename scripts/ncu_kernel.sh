#!/bin/bash
# usage: scripts/ncu_kernel.sh <out-name> <kernel-regex> <solver> [config]
# One --set full capture of the first launch of <kernel-regex> in scripts/prof_solver.py.
set -e
out=$1; kre=$2; solver=$3; cfg=${4:-C}
python scripts/prof_solver.py --solver $solver --config $cfg --reps 1 > /dev/null
ncu --set full --import-source on --clock-control none -k regex:$kre -c 1 -o gpurun_out/$out -f \
    python scripts/prof_solver.py --solver $solver --config $cfg --reps 1 > gpurun_out/$out.log 2>&1
