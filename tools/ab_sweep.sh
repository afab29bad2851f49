#!/bin/bash
# Same-box A/B of environment settings (run on the GPU box from the repo root): each argument is a set of
# VAR=value pairs (e.g. "LG_DW1_CTAS=100" or "LG_LIB=path/to/other/libleggedrl.so"); every setting runs
# `bench.py --steps 30` twice, interleaved, and prints the ms per iteration.
# usage: tools/ab_sweep.sh "X=0" "LG_LOSS_ACTOR_FRAC=0.5" ...
mkdir -p gpurun_out/sw
for rep in 1 2; do
for s in "$@"; do
  env $s timeout 200 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/sw/tmp.txt 2>&1
  ms=$(grep '^{' gpurun_out/sw/tmp.txt | tail -1 | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['ms_per_step'],4))" 2>/dev/null)
  echo "$rep [$s] $ms" | tee -a gpurun_out/sw/result.txt
done; done
