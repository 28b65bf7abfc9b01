mkdir -p gpurun_out/sanitize
for ws in 0 1; do BE_SPMM_WS=$ws timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 10 python tools/sanitize_workload.py > gpurun_out/sanitize/racecheck2_ws$ws.log 2>&1; echo "racecheck ws=$ws rc=$?"; done
