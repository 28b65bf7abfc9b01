#!/bin/bash
# Round-2 one-GPU sweep: bench lines (jsonl) + per-phase device times (BE_TRACE_SEGMENTS) per configuration.
# Usage (on the GPU box): bash tools/sweep_r02.sh OUT_PREFIX "args1" "args2" ...
out=$1; shift
for args in "$@"; do
  tag=$(echo "$args" | tr ' -' '_' | tr -s '_')
  BE_TRACE_SEGMENTS=1 timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline $args \
     > gpurun_out/${out}${tag}.json 2> gpurun_out/${out}${tag}.err
  echo "$args rc=$?" >> gpurun_out/${out}index.txt
done
