#!/bin/bash
# Batched-decode sweep (configs[4]): one JSON line per B (sparse tcgen05 path, dense
# comparator, e2e, roofline) into gpurun_out/batch_B*.json.
#   tools/batch_sweep.sh [layers] [B ...]     (default: the full 32-layer 7B stack)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=${1:-32}; shift
for B in ${@:-2 4 8 16 32 64}; do
  python bench.py --batch $B --layers $L --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/batch_B$B.json 2> gpurun_out/batch_B$B.err
  python -c "import json; d=json.loads(open('gpurun_out/batch_B$B.json').read().strip().splitlines()[-1]); print('B=$B', 'us/layer %.1f frac %.3f | dense us/layer %.1f frac %.3f | speedup %.2f' % (d['per_layer_us'], d['roofline']['frac'], d['dense']['per_layer_us'], d['dense']['frac'], d['dense']['sparse_speedup']))" || tail -5 gpurun_out/batch_B$B.err
done
