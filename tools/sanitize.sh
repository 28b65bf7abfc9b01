#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over small shapes of every device kernel
# (run on the GPU box): SpMM (classic, warp-specialised, deterministic), preconditioner classes,
# dense panel kernels, the fused Rayleigh-Ritz eigensolve and a short LOBPCG solve.
out=${1:-gpurun_out/sanitize}
mkdir -p $out
for tool in memcheck racecheck synccheck; do
  for ws in 0 1; do
    BE_SPMM_WS=$ws timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 \
      --print-limit 20 python tools/sanitize_workload.py > $out/${tool}_ws$ws.log 2>&1
    echo "$tool ws=$ws rc=$?" >> $out/summary.txt
  done
done
cat $out/summary.txt
