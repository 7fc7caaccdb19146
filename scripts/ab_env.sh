#!/bin/bash
# Same-box A/B of an environment switch (experiments):
#   scripts/ab_env.sh TEM_NO_PAIR=1 [config tol maxit]   -> gpurun_out/abe.log
# alternates the default run and the run with the variable set, three rounds.
mkdir -p gpurun_out
var=$1; cfg=${2:-large-fit}; tol=${3:-1e-10}; maxit=${4:-2000}
for rep in 1 2 3; do
  python scripts/probe_solvers.py $cfg $tol split $maxit 2>&1 | grep -E "^split" | sed -E "s/^/$cfg default /" >> gpurun_out/abe.log
  env $var python scripts/probe_solvers.py $cfg $tol split $maxit 2>&1 | grep -E "^split" | sed -E "s/^/$cfg $var /" >> gpurun_out/abe.log
done
