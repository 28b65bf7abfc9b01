set -x
for args in "--nb 8" "--nb 16" "--nb 32" "--nb 16 --precond off" "--nb 8 --precond off" "--nb 32 --precond off" "--config c1 --nb 16"; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-gate $args 2>/dev/null | tail -n 1 >> gpurun_out/sweep2.jsonl
done
