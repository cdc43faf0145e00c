#!/bin/bash
# Batched-decode sweep (configs[4]) on the full 32-layer 7B stack: one JSON line per B
# (sparse tcgen05 path, dense comparator, e2e, roofline) into gpurun_out/batch_B*.json.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for B in ${@:-2 4 8 16 32 64}; do
  python bench.py --batch $B --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/batch_B$B.json 2> gpurun_out/batch_B$B.err
  echo "B=$B exit=$?"
done
